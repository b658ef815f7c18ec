// lja.cuh -- shared argument plumbing and validation of the lifted join-aggregate kernels.
#pragma once
#include "segwalk.cuh"

namespace rnn {

struct OpndD {
  const float* p;
  int64_t ld;
  int dim;
  int mode;
};

// node epilogue (rnn_epilogue) in device form: y = gate * act(x + bias) + (1 - gate) * resid
struct EpiD {
  int on;
  const float* bias;
  int act;               // 0 none, 1 ReLU, 2 GELU
  float gate;
  const float* resid;
  int64_t ld_resid;
  float* pre;
  int64_t ld_pre;
};

__device__ __forceinline__ float epi_act(int act, float x) {
  if (act == 1) return fmaxf(x, 0.f);
  if (act == 2) return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
  return x;
}
__device__ __forceinline__ float epi_dact(int act, float x) {   // d act / dx at x
  if (act == 1) return x > 0.f ? 1.f : 0.f;
  if (act == 2) {
    const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
    const float pdf = 0.39894228040143268f * __expf(-0.5f * x * x);
    return cdf + x * pdf;
  }
  return 1.f;
}
// the epilogue of row g, columns c .. c+3 (x already holds the aggregate)
__device__ __forceinline__ float4 epi_apply4(const EpiD& e, float4 x, int64_t g, int c) {
  if (e.bias) x = f4_add(x, *reinterpret_cast<const float4*>(e.bias + c));
  if (e.pre) *reinterpret_cast<float4*>(e.pre + g * e.ld_pre + c) = x;
  x = make_float4(epi_act(e.act, x.x), epi_act(e.act, x.y), epi_act(e.act, x.z),
                  epi_act(e.act, x.w));
  if (e.resid) {
    const float4 r = *reinterpret_cast<const float4*>(e.resid + g * e.ld_resid + c);
    const float a = e.gate;
    x = make_float4(a * x.x + (1.f - a) * r.x, a * x.y + (1.f - a) * r.y,
                    a * x.z + (1.f - a) * r.z, a * x.w + (1.f - a) * r.w);
  }
  return x;
}

struct LjaArgs {
  const int64_t* group_ptr;
  const int32_t* src_row;
  const int32_t* edge_row;
  const int32_t* dst_row;
  OpndD src, src_key, edge, dst;
  int combine;
  int mean;
  float* out;
  int64_t ld_out;
  int D;
  float beta;
  float* lse;
  EpiD epi;        // node epilogue fused into the lean store (epi.on == 0: none)
  int* epi_done;   // host flag: set when a launcher fused the epilogue
};

struct QueryInfo {
  int D;           // output width
  bool concat;     // CONCAT path (generic per-column kernel)
  int64_t pstride; // floats per partial state of the forward
};

inline OpndD opnd(const rnn_operand& o) { return OpndD{o.data, o.ld, o.dim, o.mode}; }

// floats per partial state: the flat kernel (widths > 64) stores 32 lanes x VEC float4
inline int64_t flat_pstride(int D) { return D > 64 ? (D + 127) / 128 * 128 : (D + 3) / 4 * 4; }

// 1,2,4,8,16,32 lanes per row (one float4 each), or 64 / 128 float4 columns (VEC 2 / 4)
inline int lane_config(int D) {
  const int n4 = (D + 3) / 4;
  if (n4 <= 32) {
    int l = 1;
    while (l < n4) l <<= 1;
    return l;
  }
  if (n4 <= 64) return 64;
  if (n4 <= 128) return 128;
  return 0;
}

inline rnn_status check_operand(const rnn_operand& o, const char* name, bool allow_scalar_ld) {
  if (!o.data) return RNN_OK;
  RNN_REQUIRE(o.dim >= 1 && o.dim <= 512, RNN_ERR_UNSUPPORTED, "%s.dim=%d outside [1,512]", name,
              o.dim);
  RNN_REQUIRE(o.ld >= o.dim, RNN_ERR_INVALID_ARGUMENT, "%s.ld < dim", name);
  RNN_REQUIRE(o.mode == RNN_BY_ROW || o.mode == RNN_BY_POSITION, RNN_ERR_INVALID_ARGUMENT,
              "%s.mode invalid", name);
  if (!(allow_scalar_ld && o.dim == 1))
    RNN_REQUIRE(o.ld % 4 == 0 && aligned16(o.data), RNN_ERR_INVALID_ARGUMENT,
                "%s must be 16-byte aligned with ld %% 4 == 0", name);
  return RNN_OK;
}

inline rnn_status check_query(const rnn_join_index* idx, const rnn_lifted_query* q,
                              QueryInfo* qi) {
  RNN_REQUIRE(idx && q, RNN_ERR_INVALID_ARGUMENT, "idx and q are required");
  RNN_REQUIRE(idx->group_ptr && (idx->n_groups == 0 || (idx->src_row && idx->edge_row &&
                                                        idx->group_dst_row && idx->work_ptr)),
              RNN_ERR_INVALID_ARGUMENT, "index arrays missing (build the index first)");
  RNN_TRY(check_operand(q->src, "src", false));
  RNN_TRY(check_operand(q->src_key, "src_key", false));
  RNN_TRY(check_operand(q->edge, "edge", true));
  RNN_TRY(check_operand(q->dst, "dst", true));
  const bool hs = q->src.data, hk = q->src_key.data, he = q->edge.data, ht = q->dst.data;
  RNN_REQUIRE(!hs || q->src.mode == RNN_BY_ROW, RNN_ERR_UNSUPPORTED, "src must use RNN_BY_ROW");
  RNN_REQUIRE(!(hs || hk) || idx->n_src_rows > 0 || idx->n_groups == 0, RNN_ERR_INVALID_ARGUMENT,
              "src operand given but the index has no S relation");
  RNN_REQUIRE(!ht || q->dst.mode == RNN_BY_POSITION || idx->n_dst_rows > 0 || idx->n_groups == 0,
              RNN_ERR_INVALID_ARGUMENT, "dst operand by row but the index has no T relation");
  qi->concat = false;
  if (q->agg == RNN_AGG_SOFTMAX) {
    RNN_REQUIRE(q->combine == RNN_COMBINE_SRC, RNN_ERR_UNSUPPORTED, "SOFTMAX needs combine SRC");
    RNN_REQUIRE(hs && hk && ht && !he, RNN_ERR_INVALID_ARGUMENT,
                "SOFTMAX needs src (values), src_key (keys), dst (queries) and no edge");
    const int D = q->src.dim;
    RNN_REQUIRE(q->src_key.dim == D && q->dst.dim == D, RNN_ERR_SHAPE_MISMATCH,
                "SOFTMAX needs src, src_key and dst of equal width");
    RNN_REQUIRE(D == 4 || D == 8 || D == 16 || D == 32 || D == 64 || D == 128, RNN_ERR_UNSUPPORTED,
                "SOFTMAX width must be a power of two in [4,128]");
    RNN_REQUIRE(q->heads >= 1 && D % q->heads == 0 && (D / q->heads) % 4 == 0,
                RNN_ERR_UNSUPPORTED, "heads must divide width with width/heads %% 4 == 0");
    RNN_REQUIRE(q->dst.dim > 1, RNN_ERR_UNSUPPORTED, "queries must be vectors");
    qi->D = D;
    qi->pstride = (D + 2 * q->heads + 3) / 4 * 4;
    return RNN_OK;
  }
  RNN_REQUIRE(q->agg == RNN_AGG_SUM || q->agg == RNN_AGG_MEAN, RNN_ERR_INVALID_ARGUMENT,
              "agg invalid");
  switch (q->combine) {
    case RNN_COMBINE_SRC:
      RNN_REQUIRE(hs && !ht && !hk, RNN_ERR_INVALID_ARGUMENT,
                  "combine SRC needs src and no dst/src_key");
      RNN_REQUIRE(!he || q->edge.dim == 1, RNN_ERR_SHAPE_MISMATCH,
                  "combine SRC takes a scalar (dim 1) edge weight");
      qi->D = q->src.dim;
      break;
    case RNN_COMBINE_MUL:
    case RNN_COMBINE_ADD: {
      RNN_REQUIRE(!hk, RNN_ERR_INVALID_ARGUMENT, "src_key only for SOFTMAX");
      RNN_REQUIRE(hs || he || ht, RNN_ERR_INVALID_ARGUMENT, "no operand");
      int D = 0;
      if (hs) D = q->src.dim;
      if (he && q->edge.dim > D) D = q->edge.dim;
      if (ht && q->dst.dim > D) D = q->dst.dim;
      RNN_REQUIRE(!hs || q->src.dim == D, RNN_ERR_SHAPE_MISMATCH, "src.dim must equal the width");
      RNN_REQUIRE(!he || q->edge.dim == D || q->edge.dim == 1, RNN_ERR_SHAPE_MISMATCH,
                  "edge.dim must be 1 or the width");
      RNN_REQUIRE(!ht || q->dst.dim == D || q->dst.dim == 1, RNN_ERR_SHAPE_MISMATCH,
                  "dst.dim must be 1 or the width");
      qi->D = D;
      break;
    }
    case RNN_COMBINE_CONCAT:
      RNN_REQUIRE(!hk, RNN_ERR_INVALID_ARGUMENT, "src_key only for SOFTMAX");
      RNN_REQUIRE(hs || he || ht, RNN_ERR_INVALID_ARGUMENT, "no operand");
      qi->D = (hs ? q->src.dim : 0) + (he ? q->edge.dim : 0) + (ht ? q->dst.dim : 0);
      RNN_REQUIRE(qi->D <= 512, RNN_ERR_UNSUPPORTED, "CONCAT width %d > 512", qi->D);
      qi->concat = true;
      break;
    default:
      RNN_FAIL(RNN_ERR_INVALID_ARGUMENT, "combine invalid");
  }
  RNN_REQUIRE(lane_config(qi->D) != 0, RNN_ERR_UNSUPPORTED, "width %d > 512", qi->D);
  qi->pstride = flat_pstride(qi->D);
  return RNN_OK;
}

inline LjaArgs make_args(const rnn_join_index* idx, const rnn_lifted_query* q, float* out,
                         int64_t ld_out, float beta, float* lse, int D) {
  LjaArgs a{};
  a.group_ptr = idx->group_ptr;
  a.src_row = idx->src_row;
  a.edge_row = idx->edge_row;
  a.dst_row = idx->group_dst_row;
  a.src = opnd(q->src);
  a.src_key = opnd(q->src_key);
  a.edge = opnd(q->edge);
  a.dst = opnd(q->dst);
  a.combine = q->combine;
  a.mean = q->agg == RNN_AGG_MEAN;
  a.out = out;
  a.ld_out = ld_out;
  a.D = D;
  a.beta = beta;
  a.lse = lse;
  return a;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline rnn_status lja_fwd_ws(const rnn_join_index* idx, const rnn_lifted_query* q, size_t* b) {
  QueryInfo qi;
  RNN_TRY(check_query(idx, q, &qi));
  *b = qi.concat ? 0
                 : align256(sizeof(float) * idx->n_work * qi.pstride) +
                       align256(sizeof(int) * idx->n_work) + 512;
  return RNN_OK;
}

rnn_status lja_fwd_impl(const rnn_join_index* idx, const rnn_lifted_query* q, float* out,
                        int64_t ld_out, float beta, float* lse, void* ws, size_t ws_bytes,
                        cudaStream_t st,
                        const EpiD* epi = nullptr);
rnn_status epilogue_inplace(float* y, int64_t ldy, int64_t rows, int dim, const EpiD& e,
                            cudaStream_t st);
EpiD epi_from_abi(const rnn_epilogue* e);
rnn_status lja_bwd_ws(const rnn_join_index* idx, const rnn_lifted_query* q, size_t* b);

}  // namespace rnn
