// project.cu -- A2: the dense per-relation projection Y = X W^T + b on tcgen05 tensor cores.
//
// This is the transformation T_tau pushed below the join so it runs once per node instead of
// once per edge (the paper's physical plan applies nn.Linear).
//
// Kernel anatomy (one 128-row output tile per CTA, 192 threads, warp-specialised):
//   warp 0      : TMA producer -- cp.async.bulk.tensor 2D boxes into a STAGES-deep ring of
//                 128B-swizzled shared-memory tiles, signalling `full` mbarriers (complete_tx).
//   warp 1      : allocates TMEM, one elected lane issues tcgen05.mma.kind::tf32 (M=128,
//                 N=BN, K=8 per instruction) from smem descriptors, accumulating in TMEM;
//                 tcgen05.commit frees each stage (`empty`) and finally signals `acc_full`.
//   warps 2..5  : 3xTF32 only: split every landed tile into hi = tf32(x) and lo = x - hi
//                 (so the MMA computes hi*hi + hi*lo + lo*hi ~ fp32 accuracy); then the
//                 epilogue: tcgen05.ld 32x32b TMEM -> registers, + bias, store.
// Operands may be K-major (row-major [rows, K]) or MN-major (row-major [K, rows]) -- the
// latter gives dW = dY^T X without materialising transposes (smem descriptor major bit).
// Split-K over z with partial tiles reduced in a fixed order keeps dW deterministic.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace rnn {
namespace {

constexpr int BM = 128;   // UMMA_M (cta_group::1): accumulator row i <-> TMEM lane i
constexpr int BK = 32;    // fp32 elements per 128-byte swizzle row
constexpr int THREADS = 320;    // tile GEMM: producer, MMA, 8 converter warps (2-9; 2-5 epilogue)
constexpr int CONV_THREADS = 256;
constexpr int MAX_STAGES = 8;

struct GemmParams {
  int64_t M;        // output rows
  int N;            // output cols
  int BN;           // tile cols (multiple of 16 (K-major B) or 32 (MN-major B))
  int64_t Kred;     // reduction length
  int64_t k_split;  // reduction elements per blockIdx.z (multiple of BK)
  int stages;
  float* out; int64_t ldo;
  const float* bias;
  int mode;         // 0: out = acc + bias ; 1: partial[z] = acc
  float* partial; int64_t ldp; int64_t part_stride;
  uint32_t tmem_cols;
  int a3d, b3d;     // MN-major operand loaded as ONE 3D box {32, KB, MN/32} per stage
  int smem_kb;      // shared-memory budget of the stage ring (0: default 200 KB, 1 CTA / SM)
  int b_lo_row;     // K-major B with its 3xTF32 lo part precomputed b_lo_row rows below (0: none)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, void* dst, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, void* dst, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor (sm_100 version bits = 1).
//  K-major : SWIZZLE_128B (layout type 2): 8-row x 128B atoms stacked every 1024B (SBO); the
//            K step of 8 tf32 elements is a 32-byte advance of the start address.
//  MN-major: tf32 (32-bit) MN-major operands only support SWIZZLE_128B_BASE32B (layout type
//            1): atoms of 32 MN elements (128B) x 4 K-rows with 32-byte chunks swizzled by
//            the K row (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B); 32-wide MN chunks every
//            `lbo` bytes (LBO), 4-row K groups every 512B (SBO); the K step of 8 rows is a
//            1024-byte advance.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, bool mn_major, int kk, uint32_t lbo) {
  const uint32_t start = saddr + (mn_major ? kk * 1024u : kk * 32u);
  const uint64_t LBO = mn_major ? (lbo >> 4) : 1u;
  const uint64_t SBO = mn_major ? (512u >> 4) : (1024u >> 4);
  const uint64_t layout = mn_major ? 1ull : 2ull;
  return (uint64_t)((start >> 4) & 0x3FFFu) | ((LBO & 0x3FFFull) << 16) |
         ((SBO & 0x3FFFull) << 32) | (1ull << 46) | (layout << 61);
}

// Instruction descriptor for kind::tf32: D=F32, A=B=TF32, M=128, N=bn.
__device__ __forceinline__ uint32_t make_idesc(int bn, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// lo = x - trunc_tf32(x) only: the tcgen05 tf32 MMA truncates its fp32 inputs itself, so the
// raw tile is its own hi part
__device__ __forceinline__ float4 lo_part(float4 v) {
  float4 l;
  l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
  l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
  l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
  l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
  return l;
}
// NT threads; 8 shared-memory loads in flight per thread (the converter was latency-bound)
template <int NT = 128>
__device__ __forceinline__ void lo_tile(const float4* x, float4* lo, uint32_t n16, int t) {
  uint32_t i = t;
  for (; i + 7 * NT < n16; i += 8 * NT) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = x[i + u * NT];
#pragma unroll
    for (int u = 0; u < 8; ++u) lo[i + u * NT] = lo_part(v[u]);
  }
  for (; i < n16; i += NT) lo[i] = lo_part(x[i]);
}

// RNN_PREC_BF16: operands rounded to bf16 (round-to-nearest-even) in shared memory; a bf16 value
// is exact in tf32 (8-bit exponent, 7 <= 10 mantissa bits), so the kind::tf32 MMA then forms the
// exact bf16 x bf16 products with fp32 accumulation -- numerically a bf16 GEMM over fp32 storage
__device__ __forceinline__ float bf16_rn(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float4 bf16_rn4(float4 v) {
  return make_float4(bf16_rn(v.x), bf16_rn(v.y), bf16_rn(v.z), bf16_rn(v.w));
}
template <int NT = 128>
__device__ __forceinline__ void bf16_tile(float4* x, uint32_t n16, int t) {
  uint32_t i = t;
  for (; i + 7 * NT < n16; i += 8 * NT) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = x[i + u * NT];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[i + u * NT] = bf16_rn4(v[u]);
  }
  for (; i < n16; i += NT) x[i] = bf16_rn4(x[i]);
}

// precision modes of the tensor-core kernels (template argument PM = rnn_precision)
constexpr int PM_TF32 = 0, PM_3X = 1, PM_BF16 = 2;

// per-role wait cycles of tc_gemm_kernel (internal hook rnn_internal_gemm_stats): [0] producer
// waits for a free slot, [1] MMA waits for a ready stage, [2] converter waits for a landed
// stage, [3] TMA latency (issue -> landed, summed over stages, converter / MMA side),
// [4] stages counted for [3]; [8..10] total cycles of producer, MMA, converter lanes
__device__ unsigned long long g_gemm_stats[16];

template <bool A_MN, bool B_MN, int PM, int KB = BK>
__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   GemmParams p) {
  constexpr bool SPLIT3 = PM == PM_3X;   // hi/lo split tiles
  constexpr bool CONV = PM != PM_TF32;   // a converter pass over every landed stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte align the carve (swizzle atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  // KB = reduction elements per stage: 32 (K-major, one 128-byte swizzle row) or 16 (MN-major
  // operands: half-size stages, twice as many in flight)
  const uint32_t A_BYTES = BM * KB * 4;
  const uint32_t B_BYTES = (uint32_t)p.BN * KB * 4;
  const uint32_t STAGE = (A_BYTES + B_BYTES) * (SPLIT3 ? 2u : 1u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * STAGE);
  uint64_t* empty = full + MAX_STAGES;
  uint64_t* conv = empty + MAX_STAGES;
  uint64_t* acc_full = conv + MAX_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RNN_PROBE(const long long gs_t0 = clock64(); unsigned long long gs_w[5] = {0, 0, 0, 0, 0};
            __shared__ long long gs_issue[MAX_STAGES];)
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * p.BN;
  const int64_t kbeg = (int64_t)blockIdx.z * p.k_split;
  const int64_t kend = kbeg + p.k_split < p.Kred ? kbeg + p.k_split : p.Kred;
  const int nkb = (int)((kend - kbeg + KB - 1) / KB);

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < MAX_STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
        mbar_init(&conv[s], CONV_THREADS);
      }
      mbar_init(acc_full, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto a_hi = [&](int s) { return smem + s * STAGE; };
  auto b_hi = [&](int s) { return smem + s * STAGE + A_BYTES; };
  auto a_lo = [&](int s) { return smem + s * STAGE + A_BYTES + B_BYTES; };
  auto b_lo = [&](int s) { return smem + s * STAGE + 2 * A_BYTES + B_BYTES; };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % p.stages;
        const uint32_t ph = (kb / p.stages) & 1;
        if (kb >= p.stages) {
          RNN_PROBE(const long long t0 = clock64();)
          mbar_wait(&empty[s], ph ^ 1);
          RNN_PROBE(gs_w[0] += clock64() - t0;)
        }
        RNN_PROBE(gs_issue[s] = clock64();)
        const bool blo = SPLIT3 && !B_MN && p.b_lo_row > 0;
        mbar_expect_tx(&full[s], A_BYTES + B_BYTES * (blo ? 2u : 1u));
        const int k = (int)(kbeg + (int64_t)kb * KB);
        // MN-major operands: 32-wide MN chunks every KB * 128 bytes, either one 3D box
        // {32, KB, chunks} (a single TMA op) or one 2D box per chunk
        if (!A_MN) {
          tma_load_2d(&ta, a_hi(s), &full[s], k, (int)m0);
        } else if (p.a3d) {
          tma_load_3d(&ta, a_hi(s), &full[s], 0, k, (int)(m0 / 32));
        } else {
#pragma unroll
          for (int j = 0; j < BM / 32; ++j)
            tma_load_2d(&ta, a_hi(s) + j * (KB * 128), &full[s], (int)m0 + 32 * j, k);
        }
        if (!B_MN) {
          tma_load_2d(&tb, b_hi(s), &full[s], k, n0);
          if (blo) tma_load_2d(&tb, b_lo(s), &full[s], k, n0 + p.b_lo_row);
        } else if (p.b3d) {
          tma_load_3d(&tb, b_hi(s), &full[s], 0, k, n0 / 32);
        } else {
          for (int j = 0; j < p.BN / 32; ++j)
            tma_load_2d(&tb, b_hi(s) + j * (KB * 128), &full[s], n0 + 32 * j, k);
        }
      }
      RNN_PROBE(atomicAdd(&g_gemm_stats[8], (unsigned long long)(clock64() - gs_t0));
                atomicAdd(&g_gemm_stats[0], gs_w[0]);)
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc(p.BN, A_MN, B_MN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % p.stages;
      const uint32_t ph = (kb / p.stages) & 1;
      {
        RNN_PROBE(const long long t0 = clock64();)
        mbar_wait(CONV ? &conv[s] : &full[s], ph);
        RNN_PROBE(const long long t1 = clock64(); gs_w[1] += t1 - t0;
                  if (!SPLIT3) { gs_w[3] += t1 - *(volatile long long*)&gs_issue[s]; gs_w[4] += 1; })
      }
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < KB / 8; ++kk) {
          const uint64_t ad = make_desc(smem_u32(a_hi(s)), A_MN, kk, KB * 128);
          const uint64_t bd = make_desc(smem_u32(b_hi(s)), B_MN, kk, KB * 128);
          tc_mma_tf32(tmem, ad, bd, idesc, (kb | kk) != 0);
          if (SPLIT3) {
            const uint64_t al = make_desc(smem_u32(a_lo(s)), A_MN, kk, KB * 128);
            const uint64_t bl = make_desc(smem_u32(b_lo(s)), B_MN, kk, KB * 128);
            tc_mma_tf32(tmem, ad, bl, idesc, 1u);
            tc_mma_tf32(tmem, al, bd, idesc, 1u);
          }
        }
        tc_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) tc_commit(acc_full);
    __syncwarp();
    RNN_PROBE(if (lane == 0) {
      atomicAdd(&g_gemm_stats[9], (unsigned long long)(clock64() - gs_t0));
      atomicAdd(&g_gemm_stats[1], gs_w[1]);
      if (!SPLIT3) { atomicAdd(&g_gemm_stats[3], gs_w[3]); atomicAdd(&g_gemm_stats[4], gs_w[4]); }
    })
  } else {
    // ---------------- converters (3xTF32): warps 2..9; epilogue: warps 2..5 ----------------
    const int et = threadIdx.x - 64;  // 0..255
    if (CONV) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % p.stages;
        const uint32_t ph = (kb / p.stages) & 1;
        {
          RNN_PROBE(const long long t0 = clock64();)
          mbar_wait(&full[s], ph);
          RNN_PROBE(const long long t1 = clock64(); gs_w[2] += t1 - t0;
                    gs_w[3] += t1 - *(volatile long long*)&gs_issue[s]; gs_w[4] += 1;)
        }
        if (SPLIT3) {
          // lo = x - trunc_tf32(x); the raw tile is the hi part (the MMA truncates)
          lo_tile<CONV_THREADS>(reinterpret_cast<const float4*>(a_hi(s)),
                                reinterpret_cast<float4*>(a_lo(s)), A_BYTES / 16, et);
          if (B_MN || p.b_lo_row == 0)   // else B's lo part was precomputed and loaded by TMA
            lo_tile<CONV_THREADS>(reinterpret_cast<const float4*>(b_hi(s)),
                                  reinterpret_cast<float4*>(b_lo(s)), B_BYTES / 16, et);
        } else {
          bf16_tile<CONV_THREADS>(reinterpret_cast<float4*>(a_hi(s)), A_BYTES / 16, et);
          bf16_tile<CONV_THREADS>(reinterpret_cast<float4*>(b_hi(s)), B_BYTES / 16, et);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&conv[s]);
      }
    }
    RNN_PROBE(if (lane == 0 && warp == 2) {
      atomicAdd(&g_gemm_stats[10], (unsigned long long)(clock64() - gs_t0));
      for (int i = 2; i < 5; ++i) atomicAdd(&g_gemm_stats[i], gs_w[i]);
    })
    if (warp < 6) mbar_wait(acc_full, 0);   // warps 6-9 only convert
    tc_fence_after();
    const int quad = warp & 3;  // TMEM lanes [32*quad, 32*quad+32) belong to this warp
    const int64_t row = m0 + quad * 32 + lane;
    const bool row_ok = row < p.M;
    for (int c0 = 0; c0 < (warp < 6 ? p.BN : 0); c0 += 16) {
      uint32_t r[16];
      tc_ld16(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0, r);
      if (!row_ok) continue;
      const int col0 = n0 + c0;
      if (p.mode == 0) {
        float* dst = p.out + row * p.ldo + col0;
        const bool vec = col0 + 16 <= p.N && (p.ldo % 4 == 0) &&
                         ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0);
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          v[j] = __uint_as_float(r[j]) + ((p.bias && col0 + j < p.N) ? __ldg(p.bias + col0 + j) : 0.f);
        if (vec) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (col0 + j < p.N) dst[j] = v[j];
        }
      } else {
        float* dst = p.partial + blockIdx.z * p.part_stride + row * p.ldp + col0;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (col0 + j < p.N) dst[j] = __uint_as_float(r[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(p.tmem_cols));
  }
}

// ------------------------------------------------------------------------------------------
// Persistent projection kernel: Y[M, N] = A[M, K] B[N, K]^T (+ bias), both K-major, for the
// tall-skinny shapes of the hot path (M = node count, K, N <= a few hundred).  The operand B
// (the weight tile of this CTA's column block) is loaded ONCE and stays resident in shared
// memory (split into hi/lo once for 3xTF32); the CTA then streams 128-row tiles of A through a
// TMA ring, accumulating into one of two TMEM buffers while dedicated epilogue warps drain the
// other, so loads, MMAs and stores of consecutive tiles overlap.  One CTA per SM; CTA c owns
// column block c % n_tiles_n and row tiles c / n_tiles_n, + grid / n_tiles_n, ...
//   warp 0: TMA producer    warp 1: TMEM alloc + MMA issuer
//   warps 2-5: 3xTF32 hi/lo converters    warps 6-9: epilogue (TMEM -> registers -> HBM)
// ------------------------------------------------------------------------------------------
constexpr int PT_THREADS = 320;
constexpr int PT_MAX_STAGES = 6;

struct ProjParams {
  int64_t M;
  int N, BN, n_tiles_n;
  int64_t n_tiles_m;
  int nkb;                // K blocks of BK
  int stages;
  float* out; int64_t ldo;
  const float* bias;
  uint32_t tmem_cols;
};

__device__ __forceinline__ void split_tile(float4* hi, float4* lo, uint32_t n16, int t) {
  for (uint32_t i = t; i < n16; i += 128) {
    float4 x = hi[i], h, l;
    h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u); l.x = x.x - h.x;
    h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u); l.y = x.y - h.y;
    h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u); l.z = x.z - h.z;
    h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u); l.w = x.w - h.w;
    hi[i] = h; lo[i] = l;
  }
}

template <int PM>
__global__ void __launch_bounds__(PT_THREADS, 1)
    tc_proj_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   ProjParams p) {
  constexpr bool SPLIT3 = PM == PM_3X, CONV = PM != PM_TF32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr uint32_t A_BYTES = BM * BK * 4;
  const uint32_t B_BYTES = (uint32_t)p.BN * BK * 4;            // one K block of B
  const uint32_t B_RES = B_BYTES * p.nkb;                       // resident B (hi)
  const uint32_t A_STAGE = A_BYTES * (SPLIT3 ? 2u : 1u);
  uint8_t* b_hi = smem;
  uint8_t* b_lo = smem + B_RES;
  uint8_t* a_base = smem + B_RES * (SPLIT3 ? 2u : 1u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(a_base + p.stages * A_STAGE);
  uint64_t* a_full = bars;
  uint64_t* a_conv = a_full + PT_MAX_STAGES;
  uint64_t* a_empty = a_conv + PT_MAX_STAGES;
  uint64_t* b_full = a_empty + PT_MAX_STAGES;
  uint64_t* b_conv = b_full + 1;
  uint64_t* acc_full = b_conv + 1;     // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = blockIdx.x % p.n_tiles_n;
  const int n0 = nt * p.BN;
  const int64_t mt0 = blockIdx.x / p.n_tiles_n;
  const int64_t mstep = gridDim.x / p.n_tiles_n;

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < PT_MAX_STAGES; ++s) {
        mbar_init(&a_full[s], 1);
        mbar_init(&a_conv[s], 128);
        mbar_init(&a_empty[s], 1);
      }
      mbar_init(b_full, 1);
      mbar_init(b_conv, 128);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&acc_full[b], 1);
        mbar_init(&acc_empty[b], 128);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(b_full, B_RES);
      for (int kb = 0; kb < p.nkb; ++kb) tma_load_2d(&tb, b_hi + kb * B_BYTES, b_full, kb * BK, n0);
      int64_t it = 0;
      for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep) {
        for (int kb = 0; kb < p.nkb; ++kb, ++it) {
          const int s = (int)(it % p.stages);
          const uint32_t ph = (uint32_t)((it / p.stages) & 1);
          if (it >= p.stages) mbar_wait(&a_empty[s], ph ^ 1);
          mbar_expect_tx(&a_full[s], A_BYTES);
          tma_load_2d(&ta, a_base + s * A_STAGE, &a_full[s], kb * BK, (int)(mt * BM));
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(p.BN, false, false);
    mbar_wait(CONV ? b_conv : b_full, 0);
    tc_fence_after();
    int64_t it = 0;
    int j = 0;
    for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep, ++j) {
      const int buf = j & 1;
      if (j >= 2) mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(buf * p.BN);
      for (int kb = 0; kb < p.nkb; ++kb, ++it) {
        const int s = (int)(it % p.stages);
        const uint32_t ph = (uint32_t)((it / p.stages) & 1);
        mbar_wait(CONV ? &a_conv[s] : &a_full[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ah = smem_u32(a_base + s * A_STAGE);
          const uint32_t bh = smem_u32(b_hi + kb * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t ad = make_desc(ah, false, kk, 0);
            const uint64_t bd = make_desc(bh, false, kk, 0);
            tc_mma_tf32(d, ad, bd, idesc, (kb | kk) != 0);
            if (SPLIT3) {
              const uint64_t al = make_desc(ah + A_BYTES, false, kk, 0);
              const uint64_t bl = make_desc(smem_u32(b_lo + kb * B_BYTES), false, kk, 0);
              tc_mma_tf32(d, ad, bl, idesc, 1u);
              tc_mma_tf32(d, al, bd, idesc, 1u);
            }
          }
          tc_commit(&a_empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(&acc_full[buf]);
      __syncwarp();
    }
  } else if (warp < 6) {
    if (CONV) {
      const int t = threadIdx.x - 64;
      mbar_wait(b_full, 0);
      if (SPLIT3)
        split_tile(reinterpret_cast<float4*>(b_hi), reinterpret_cast<float4*>(b_lo), B_RES / 16, t);
      else
        bf16_tile(reinterpret_cast<float4*>(b_hi), B_RES / 16, t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(b_conv);
      int64_t it = 0;
      for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep) {
        for (int kb = 0; kb < p.nkb; ++kb, ++it) {
          const int s = (int)(it % p.stages);
          const uint32_t ph = (uint32_t)((it / p.stages) & 1);
          mbar_wait(&a_full[s], ph);
          uint8_t* a = a_base + s * A_STAGE;
          if (SPLIT3)
            split_tile(reinterpret_cast<float4*>(a), reinterpret_cast<float4*>(a + A_BYTES),
                       A_BYTES / 16, t);
          else
            bf16_tile(reinterpret_cast<float4*>(a), A_BYTES / 16, t);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&a_conv[s]);
        }
      }
    }
  } else {
    // epilogue warps 6..9 -> TMEM lane quadrants 2, 3, 0, 1
    const int quad = warp & 3;
    int j = 0;
    for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep, ++j) {
      const int buf = j & 1;
      mbar_wait(&acc_full[buf], (j >> 1) & 1);
      tc_fence_after();
      const int64_t row = mt * BM + quad * 32 + lane;
      const bool row_ok = row < p.M;
      float* dst_row = p.out + row * p.ldo;
      for (int c0 = 0; c0 < p.BN; c0 += 16) {
        uint32_t r[16];
        tc_ld16(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * p.BN + c0), r);
        const int col0 = n0 + c0;
        if (!row_ok || col0 >= p.N) continue;
        float v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          v[q] = __uint_as_float(r[q]) + ((p.bias && col0 + q < p.N) ? __ldg(p.bias + col0 + q) : 0.f);
        float* dst = dst_row + col0;
        if (col0 + 16 <= p.N && (p.ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            __stcs(reinterpret_cast<float4*>(dst + q), make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]));
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (col0 + q < p.N) dst[q] = v[q];
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(p.tmem_cols));
  }
}

// ------------------------------------------------------------------------------------------
// Transposed persistent projection: Y^T[n0:n0+128, tile] = Wb[n0:n0+128, :K] . X_tile^T, i.e.
// Y[M, N] = X[M, K] W[N, K]^T computed with the WEIGHT block as the MMA A operand resident in
// TMEM (tcgen05.mma A-from-TMEM: lane = output feature, column = k) and the streamed X row
// tile as the K-major B operand in shared memory.  Shared memory then holds only the X ring
// (up to 6 stages of raw 16 KB + its 3xTF32 low part), the accumulator lane is an output
// FEATURE and its columns are tile ROWS, so the epilogue's tcgen05.ld hands a warp 32
// consecutive features of one row: every global store is one coalesced 128-byte line.
// TMEM: [0, 256) two 128-column accumulators, [256, 384) W hi, [384, 512) W lo.
// Requires K <= 128 (W block hi + lo fit TMEM); N is covered by 128-feature column blocks.
//   warp 0: TMA producer   warp 1: TMEM alloc + MMA issuer   warps 2-5: X hi/lo split
//   warps 6-9: W -> TMEM (once), then the epilogue (TMEM -> registers -> HBM)
// ------------------------------------------------------------------------------------------
constexpr int PX_STAGES = 6;

// per-role wait cycles of tc_projt_kernel (lane 0 of warps 0, 1, 2, 6), read by the internal
// hook rnn_internal_proj_stats: [0] producer waits for a free slot, [1] MMA waits for W in
// TMEM, [2] MMA waits for a free accumulator, [3] MMA waits for a converted stage,
// [4] converter waits for a landed stage, [5] epilogue waits for an accumulator;
// [8..11] total cycles of the producer, MMA, converter, epilogue lanes
__device__ unsigned long long g_proj_stats[16];
#ifdef RNN_PROBES
#define PT_WAIT(slot, stmt)                                      \
  do {                                                           \
    const long long t0_ = clock64();                             \
    stmt;                                                        \
    if (lane == 0) pt_w[slot] += (unsigned long long)(clock64() - t0_); \
  } while (0)
#else
#define PT_WAIT(slot, stmt) \
  do {                      \
    stmt;                   \
  } while (0)
#endif

struct ProjTParams {
  int64_t M;            // rows of X / Y
  int N, K;             // out features, reduction length (K <= 128)
  int nkb;              // K blocks of BK (the B tile ring steps per row tile)
  int n_tiles_n;        // 128-feature column blocks
  int64_t n_tiles_m;
  int stages;
  const float* W; int64_t ldw;   // [N, K] row-major
  float* out; int64_t ldo;
  const float* bias;
  // fused ReLU backward of the layer that produced the GEMM's reduction input (dX of a
  // projection whose input X = ReLU(pre)): out *= [relu_src > 0], per-CTA column sums of the
  // masked output into colsum[blockIdx.x][N] (the producing epilogue's bias gradient)
  const float* relu_src; int64_t ld_relu;
  float* colsum;
};

__device__ __forceinline__ void tc_mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

template <int PM>
__global__ void __launch_bounds__(PT_THREADS, 1)
    tc_projt_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap ty,
                    ProjTParams p) {
  constexpr bool SPLIT3 = PM == PM_3X, CONV = PM != PM_TF32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr uint32_t X_BYTES = BM * BK * 4;             // one 128-row x 32-k block
  constexpr uint32_t X_STAGE = X_BYTES * (SPLIT3 ? 2u : 1u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.stages * X_STAGE);
  uint64_t* x_full = bars;
  uint64_t* x_conv = x_full + PX_STAGES;
  uint64_t* x_empty = x_conv + PX_STAGES;
  uint64_t* w_ready = x_empty + PX_STAGES;
  uint64_t* acc_full = w_ready + 1;    // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RNN_PROBE(const long long pt_t0 = clock64(); unsigned long long pt_w[6] = {0, 0, 0, 0, 0, 0};)
  const int nt = blockIdx.x % p.n_tiles_n;
  const int n0 = nt * 128;
  const int64_t mt0 = blockIdx.x / p.n_tiles_n;
  const int64_t mstep = gridDim.x / p.n_tiles_n;
  constexpr uint32_t W_HI = 256, W_LO = 384;

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < PX_STAGES; ++s) {
        mbar_init(&x_full[s], 1);
        mbar_init(&x_conv[s], 128);
        mbar_init(&x_empty[s], 1);
      }
      mbar_init(w_ready, 128);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&acc_full[b], 1);
        mbar_init(&acc_empty[b], 128);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep) {
        for (int kb = 0; kb < p.nkb; ++kb, ++it) {
          const int s = (int)(it % p.stages);
          const uint32_t ph = (uint32_t)((it / p.stages) & 1);
          if (it >= p.stages) PT_WAIT(0, mbar_wait(&x_empty[s], ph ^ 1));
          mbar_expect_tx(&x_full[s], X_BYTES);
          tma_load_2d(&tx, smem + s * X_STAGE, &x_full[s], kb * BK, (int)(mt * BM));
        }
      }
    }
  } else if (warp == 1) {
    // A = W block from TMEM (M = 128 features), B = X tile (N = 128 rows, K-major)
    const uint32_t idesc = make_idesc(BM, false, false);
    PT_WAIT(1, mbar_wait(w_ready, 0));
    tc_fence_after();
    int64_t it = 0;
    int j = 0;
    for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep, ++j) {
      const int buf = j & 1;
      if (j >= 2) PT_WAIT(2, mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1));
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(buf * 128);
      for (int kb = 0; kb < p.nkb; ++kb, ++it) {
        const int s = (int)(it % p.stages);
        const uint32_t ph = (uint32_t)((it / p.stages) & 1);
        PT_WAIT(3, mbar_wait(CONV ? &x_conv[s] : &x_full[s], ph));
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xs = smem_u32(smem + s * X_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t bh = make_desc(xs, false, kk, 0);
            const uint32_t ah = tmem + W_HI + (uint32_t)(kb * BK + kk * 8);
            tc_mma_tf32_ta(d, ah, bh, idesc, (kb | kk) != 0);
            if (SPLIT3) {
              const uint64_t bl = make_desc(xs + X_BYTES, false, kk, 0);
              tc_mma_tf32_ta(d, ah, bl, idesc, 1u);
              tc_mma_tf32_ta(d, tmem + W_LO + (uint32_t)(kb * BK + kk * 8), bh, idesc, 1u);
            }
          }
          tc_commit(&x_empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(&acc_full[buf]);
      __syncwarp();
    }
  } else if (warp < 6) {
    if (CONV) {
      const int t = threadIdx.x - 64;
      int64_t it = 0;
      for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep) {
        for (int kb = 0; kb < p.nkb; ++kb, ++it) {
          const int s = (int)(it % p.stages);
          const uint32_t ph = (uint32_t)((it / p.stages) & 1);
          PT_WAIT(4, mbar_wait(&x_full[s], ph));
          uint8_t* x = smem + s * X_STAGE;
          if (SPLIT3)
            lo_tile(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(x + X_BYTES),
                    X_BYTES / 16, t);
          else
            bf16_tile(reinterpret_cast<float4*>(x), X_BYTES / 16, t);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&x_conv[s]);
        }
      }
    }
  } else {
    const int quad = warp & 3;                 // TMEM lanes [32 quad, 32 quad + 32)
    const int f = n0 + quad * 32 + lane;       // this thread's output feature
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    // ---- W block -> TMEM (raw = hi: the MMA truncates fp32 to tf32 itself, profiles/
    // probe_tf32.py; lo = w - trunc(w)); padding features / k columns are zero.  32 x 32
    // blocks are read coalesced (lane = k) and transposed through shared memory so that
    // thread l ends up holding feature row f's k values for tcgen05.st (lane = feature).
    float* tp = reinterpret_cast<float*>(smem + p.stages * X_STAGE + 1024) + quad * 32 * 65;
    const int kpad = p.nkb * BK;
    const int fbase = n0 + quad * 32;
    const bool vec = (p.K % 4 == 0) && (p.ldw % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(p.W) & 15u) == 0);
    // 64-k halves of the warp's 32 feature rows: 16 float4 loads per thread in flight
    // (lanes 0-15 row 2rr, lanes 16-31 row 2rr+1), transposed through a [32][65] tile
    for (int k0 = 0; k0 < kpad; k0 += 64) {
      float4 v[16];
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        const int row = fbase + 2 * rr + (lane >> 4);
        const int k = k0 + 4 * (lane & 15);
        v[rr] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < p.N) {
          const float* src = p.W + (int64_t)row * p.ldw + k;
          if (vec) {
            if (k < p.K) v[rr] = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            if (k < p.K) v[rr].x = __ldg(src);
            if (k + 1 < p.K) v[rr].y = __ldg(src + 1);
            if (k + 2 < p.K) v[rr].z = __ldg(src + 2);
            if (k + 3 < p.K) v[rr].w = __ldg(src + 3);
          }
        }
      }
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        float* t = tp + (2 * rr + (lane >> 4)) * 65 + 4 * (lane & 15);
        t[0] = v[rr].x; t[1] = v[rr].y; t[2] = v[rr].z; t[3] = v[rr].w;
      }
      __syncwarp();
      for (int h = 0; h < 64 && k0 + h < kpad; h += 16) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float w = PM == PM_BF16 ? bf16_rn(tp[lane * 65 + h + q]) : tp[lane * 65 + h + q];
          hi[q] = __float_as_uint(w);
          lo[q] = __float_as_uint(w - __uint_as_float(__float_as_uint(w) & 0xFFFFE000u));
        }
        tc_st16(lane_base + W_HI + (uint32_t)(k0 + h), hi);
        if (SPLIT3) tc_st16(lane_base + W_LO + (uint32_t)(k0 + h), lo);
      }
      __syncwarp();
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    mbar_arrive(w_ready);
    // ---- epilogue ----
    // output staging (2 x 4 KB per warp) aliases the W transpose tiles, which are done
    float* stage_out = reinterpret_cast<float*>(smem + p.stages * X_STAGE + 1024) + quad * 2 * 32 * 32;
    const float bf = (p.bias && f < p.N) ? __ldg(p.bias + f) : 0.f;
    float csum = 0.f;   // fused ReLU backward: this thread's column sum (feature f)
    int j = 0;
    for (int64_t mt = mt0; mt < p.n_tiles_m; mt += mstep, ++j) {
      const int buf = j & 1;
      PT_WAIT(5, mbar_wait(&acc_full[buf], (j >> 1) & 1));
      tc_fence_after();
      const int64_t r0 = mt * BM;
      // 32-row chunks: TMEM -> registers (+bias) -> a [32 rows x 32 features] smem tile
      // (thread = feature, so each row of the tile is one conflict-free 128-byte store) ->
      // one TMA bulk tensor store; two tiles per warp alternate (wait_group.read 1)
      for (int c0 = 0; c0 < BM; c0 += 32) {
        uint32_t r[32];
        tc_ld16(lane_base + (uint32_t)(buf * 128 + c0), *reinterpret_cast<uint32_t(*)[16]>(r));
        tc_ld16(lane_base + (uint32_t)(buf * 128 + c0 + 16),
                *reinterpret_cast<uint32_t(*)[16]>(r + 16));
        // every staged chunk is committed as one bulk group, so "at most one group pending"
        // below means the previous user of this buffer has finished reading it; chunks
        // entirely outside Y are neither staged nor stored
        if (!(r0 + c0 < p.M && n0 + quad * 32 < p.N)) continue;
        const int sb = (c0 >> 5) & 1;
        float* st = stage_out + sb * 32 * 32;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        if (p.relu_src) {
          // d pre = dX (.) [X > 0]: the mask row of the producing layer's output, 32 rows per
          // chunk, each load one coalesced 128-byte row segment across the warp
          // (unpredicated loads from clamped addresses, so all 32 are in flight at once: with
          // a predicate per load the compiler ran out of predicate registers and issued each
          // load just before its use -- ncu: 483 vs 40 us per arxiv launch)
          const bool fok = f < p.N;
          const float* src = p.relu_src + (fok ? f : 0);
          float mk[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int64_t row = r0 + c0 + q;
            mk[q] = __ldg(src + (row < p.M ? row : p.M - 1) * p.ld_relu);
          }
          const int nvalid = fok ? (int)(p.M - (r0 + c0) < 32 ? p.M - (r0 + c0) : 32) : 0;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float v = (q < nvalid && mk[q] > 0.f) ? __uint_as_float(r[q]) + bf : 0.f;
            csum += v;
            st[q * 32 + lane] = v;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) st[q * 32 + lane] = __uint_as_float(r[q]) + bf;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&ty)),
              "r"(n0 + quad * 32), "r"((int)(r0 + c0)), "r"(smem_u32(st))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (p.colsum && f < p.N) p.colsum[(int64_t)blockIdx.x * p.N + f] = csum;
  }
  RNN_PROBE(if (lane == 0 && (warp == 0 || warp == 1 || warp == 2 || warp == 6)) {
    const int role = warp == 0 ? 0 : warp == 1 ? 1 : warp == 2 ? 2 : 3;
    atomicAdd(&g_proj_stats[8 + role], (unsigned long long)(clock64() - pt_t0));
    for (int i = 0; i < 6; ++i)
      if (pt_w[i]) atomicAdd(&g_proj_stats[i], pt_w[i]);
  })
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// out[i] = sum_z partial[z, i] over a contiguous [rows * cols] block, two fixed-order stages
// (deterministic split-K): blockIdx.y = g sums partials [8g, 8g + 8) into tmp[g] (float4 per
// thread, 8 loads in flight), then splitk_final sums tmp[0..G) in order.
__global__ void splitk_stage(const float* __restrict__ part, int64_t splits, int64_t stride,
                            int64_t n, float* __restrict__ tmp) {
  const int64_t i4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (4 * i4 >= n) return;
  const int64_t z0 = (int64_t)blockIdx.y * 8;
  const float4* p = reinterpret_cast<const float4*>(part) + i4;
  const int64_t s4 = stride / 4;
  float4 x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
    x[u] = z0 + u < splits ? __ldcs(p + (z0 + u) * s4) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc = x[0];
#pragma unroll
  for (int u = 1; u < 8; ++u) acc = f4_add(acc, x[u]);
  reinterpret_cast<float4*>(tmp)[blockIdx.y * (n / 4) + i4] = acc;
}
__global__ void splitk_final(const float* __restrict__ tmp, int64_t groups, int64_t n,
                             float* __restrict__ out) {
  const int64_t i4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (4 * i4 >= n) return;
  const float4* t = reinterpret_cast<const float4*>(tmp) + i4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // 8 loads in flight, additions still in group order
  for (int64_t g = 0; g < groups; g += 8) {
    float4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      x[u] = g + u < groups ? __ldcs(t + (g + u) * (n / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (g + u < groups) acc = f4_add(acc, x[u]);
  }
  reinterpret_cast<float4*>(out)[i4] = acc;
}
__global__ void splitk_reduce1(const float* __restrict__ part, int64_t splits, int64_t stride,
                               int64_t n, float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
  for (int64_t z = 0; z < splits; ++z) acc += __ldcs(part + z * stride + i);
  out[i] = acc;
}

// column sums db[c] = sum_m dY[m, c]: stage 1 (per row-chunk partials), stage 2 (ordered sum)
__global__ void colsum_partial(const float* __restrict__ Y, int64_t M, int N, int64_t ld,
                               int64_t rows_per, float* __restrict__ part) {
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int w = threadIdx.x >> 5;  // 8 warps
  __shared__ float red[8][32];
  const int64_t r0 = blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  float acc = 0.f;
  if (c < N)
    for (int64_t r = r0 + w; r < r1; r += 8) acc += Y[r * ld + c];
  red[w][threadIdx.x & 31] = acc;
  __syncthreads();
  if (w == 0) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x & 31];
    if (c < N) part[blockIdx.y * (int64_t)N + c] = s;
  }
}
// out[f] = sum_i part[(base(f) + i * stride) * N + f] over the partial rows of column f, in a
// fixed order: block = 32 columns x 8 row lanes, lane j sums rows i = j, j + 8, ... (four
// loads in flight), then the 8 lane sums are added in order (the serial one-thread-per-column
// sum was latency-bound: 22-41 us for 148-662 partial rows)
__device__ __forceinline__ void colsum8(const float* __restrict__ part, int64_t n, int64_t base,
                                        int64_t stride, int N, float* __restrict__ out) {
  __shared__ float sh[8][33];
  const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane;
  float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
  if (f < N) {
    int64_t i = j;
    for (; i + 24 < n; i += 32) {
      t0 += part[(base + i * stride) * N + f];
      t1 += part[(base + (i + 8) * stride) * N + f];
      t2 += part[(base + (i + 16) * stride) * N + f];
      t3 += part[(base + (i + 24) * stride) * N + f];
    }
    for (; i < n; i += 8) t0 += part[(base + i * stride) * N + f];
  }
  sh[j][lane] = (t0 + t1) + (t2 + t3);
  __syncthreads();
  if (j == 0 && f < N) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[q][lane];
    out[f] = s;
  }
}
__global__ void __launch_bounds__(256) colsum_final(const float* __restrict__ part, int64_t chunks,
                                                    int N, float* __restrict__ out) {
  colsum8(part, chunks, 0, 1, N, out);
}
// column sums of the fused ReLU backward (tc_projt_kernel colsum): CTA c wrote the features of
// column block c % n_tiles_n, so feature f sums the CTAs nt(f), nt(f) + n_tiles_n, ... in order
__global__ void __launch_bounds__(256) projt_colsum_final(const float* __restrict__ part, int grid,
                                                          int n_tiles_n, int N,
                                                          float* __restrict__ out) {
  const int nt = blockIdx.x * 32 / 128;   // 32-column blocks never straddle a 128-feature block
  colsum8(part, (grid - nt + n_tiles_n - 1) / n_tiles_n, nt, n_tiles_n, N, out);
}
// dX *= [X > 0] (the unfused path of rnn_project_bwd_relu)
__global__ void relu_mask_kernel(float* __restrict__ dx, int64_t lddx, const float* __restrict__ x,
                                 int64_t ldx, int64_t M, int K) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * K) return;
  const int64_t r = i / K;
  const int k = (int)(i % K);
  if (!(x[r * ldx + k] > 0.f)) dx[r * lddx + k] = 0.f;
}

// Wt[k, n] = W[n, k] (hi, rows 0..K-1) and Wt[K + k, n] = lo part (3xTF32 B operand)
__global__ void transpose_hilo_kernel(const float* __restrict__ W, int N, int K, int64_t ldw,
                                      float* __restrict__ Wt, int64_t ldt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * K) return;
  const int n = (int)(i / K), k = (int)(i % K);
  const float x = W[(int64_t)n * ldw + k];
  Wt[(int64_t)k * ldt + n] = x;
  Wt[(int64_t)(K + k) * ldt + n] = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__global__ void transpose_kernel(const float* __restrict__ W, int N, int K, int64_t ldw,
                                 float* __restrict__ Wt, int64_t ldt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * K) return;
  const int n = (int)(i / K), k = (int)(i % K);
  Wt[(int64_t)k * ldt + n] = W[(int64_t)n * ldw + k];
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D fp32 tensor [rows, inner] with row stride ld (elements); box {box_inner, box_rows}
rnn_status make_map(CUtensorMap* m, const float* base, int64_t inner, int64_t rows, int64_t ld,
                    uint32_t box_inner, uint32_t box_rows, bool mn_major = false,
                    bool swizzle = true) {
  auto fn = encode_fn();
  RNN_REQUIRE(fn, RNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  RNN_REQUIRE(aligned16(base) && (ld * 4) % 16 == 0, RNN_ERR_INVALID_ARGUMENT,
              "TMA operands need a 16-byte aligned base and ld %% 4 == 0");
  cuuint64_t dims[2] = {(cuuint64_t)(inner > 0 ? inner : 1), (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  !swizzle ? CU_TENSOR_MAP_SWIZZLE_NONE
                  : mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RNN_REQUIRE(r == CUDA_SUCCESS, RNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RNN_OK;
}

// MN-major operand [rows, mn] (row stride ld) viewed as 3D {32, rows, ceil(mn / 32)} so that one
// box {32, box_rows, chunks} lands as `chunks` 32-wide MN chunks every box_rows * 128 bytes.
// Only when the padded width fits the row stride (the last chunk's tail then reads inside the
// row; those elements only feed accumulator rows / columns >= mn, which are never stored).
bool map3_ok(const float* base, int64_t mn, int64_t ld) {
  return ld >= (mn + 31) / 32 * 32 && aligned16(base) && (ld * 4) % 16 == 0 && !getenv("RNN_NO_TMA3D");
}
rnn_status make_map3(CUtensorMap* m, const float* base, int64_t mn, int64_t rows, int64_t ld,
                     uint32_t box_rows, uint32_t chunks) {
  auto fn = encode_fn();
  RNN_REQUIRE(fn, RNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {32, (cuuint64_t)(rows > 0 ? rows : 1), (cuuint64_t)((mn + 31) / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), 128};
  cuuint32_t box[3] = {32, box_rows, chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RNN_REQUIRE(r == CUDA_SUCCESS, RNN_ERR_CUDA, "cuTensorMapEncodeTiled (3D) failed (%d)", (int)r);
  return RNN_OK;
}

uint32_t pow2_cols(int bn) {
  uint32_t c = 32;
  while ((int)c < bn) c <<= 1;
  return c;
}

template <bool A_MN, bool B_MN, int PM>
rnn_status launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, int splits,
                       cudaStream_t st) {
  constexpr bool SPLIT3 = PM == PM_3X;
  constexpr int KB = (A_MN && B_MN) ? 16 : BK;
  const uint32_t stage = (uint32_t)(BM * KB * 4 + p.BN * KB * 4) * (SPLIT3 ? 2u : 1u);
  const int64_t nkb_max = ceil_div(p.k_split, KB);
  static const int budget_kb = getenv("RNN_GEMM_SMEM_KB") ? atoi(getenv("RNN_GEMM_SMEM_KB")) : 200;
  int stages = (int)(((p.smem_kb && !getenv("RNN_GEMM_SMEM_KB") ? p.smem_kb : budget_kb) * 1024) / stage);
  if (!SPLIT3 && stages > 3 && stage * 3 <= 100 * 1024 && !(A_MN && B_MN)) stages = 3;  // 2 CTAs / SM
  if (stages > MAX_STAGES) stages = MAX_STAGES;
  if (stages > nkb_max) stages = (int)nkb_max;
  if (stages < 1) stages = 1;
  p.stages = stages;
  p.tmem_cols = pow2_cols(p.BN);
  const size_t smem = (size_t)stages * stage + 1024 + 8 * (3 * MAX_STAGES + 2) + 64;
  auto kern = tc_gemm_kernel<A_MN, B_MN, PM, KB>;
  RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)ceil_div(p.M, BM), (unsigned)ceil_div(p.N, p.BN), (unsigned)splits);
  kern<<<grid, THREADS, smem, st>>>(ta, tb, p);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

template <bool A_MN, bool B_MN>
rnn_status gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int splits,
                rnn_precision prec, cudaStream_t st) {
  if (prec == RNN_PREC_3XTF32) return launch_gemm<A_MN, B_MN, PM_3X>(ta, tb, p, splits, st);
  if (prec == RNN_PREC_BF16) return launch_gemm<A_MN, B_MN, PM_BF16>(ta, tb, p, splits, st);
  return launch_gemm<A_MN, B_MN, PM_TF32>(ta, tb, p, splits, st);
}

__global__ void bias_fill(float* Y, int64_t M, int N, int64_t ldy, const float* b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < M * N) Y[(i / N) * ldy + i % N] = b ? b[i % N] : 0.f;
}

// Fused ReLU backward for the TMEM-resident kernel (rnn_project_bwd_relu): Y *= [relu_src > 0]
// and per-CTA column sums into colsum; `fused` reports whether that kernel ran (else the caller
// masks and sums Y itself).
struct ReluBwd {
  const float* src; int64_t ld;
  float* colsum;
  bool fused; int grid, n_tiles_n;
};

// Y[M, N] = A[M, Kred] B[N, Kred]^T (+bias), both K-major
// b_has_lo: rows N .. 2N-1 of B hold lo = B - trunc_tf32(B) (precomputed by the caller)
rnn_status gemm_kk(const float* A, int64_t M, int64_t Kred, int64_t lda, const float* B, int N,
                   int64_t ldb, const float* bias, float* Y, int64_t ldy, rnn_precision prec,
                   cudaStream_t st, bool b_has_lo = false, ReluBwd* rb = nullptr) {
  if (M == 0 || N == 0) return RNN_OK;
  if (Kred == 0) {
    bias_fill<<<(unsigned)ceil_div(M * N, 256), 256, 0, st>>>(Y, M, N, ldy, bias);
    RNN_LAUNCH_CHECK();
    return RNN_OK;
  }
  if (Kred <= 128 && !getenv("RNN_NO_PROJT")) {
    // weights resident in TMEM as the A operand, X streamed as B (tc_projt_kernel)
    const bool s3 = prec == RNN_PREC_3XTF32;
    ProjTParams q{};
    q.M = M; q.N = N; q.K = (int)Kred;
    q.nkb = (int)ceil_div(Kred, BK);
    q.n_tiles_n = (int)ceil_div(N, 128);
    q.n_tiles_m = ceil_div(M, BM);
    const size_t x_stage = (size_t)BM * BK * 4 * (s3 ? 2 : 1);
    // W transpose tiles (4 x 32 x 33 floats), later the output staging (4 warps x 2 x 4 KB)
    const size_t tscratch = 4 * 2 * 32 * 32 * sizeof(float) + 1024;
    const size_t budget = 227 * 1024 - 1024 - 256 - tscratch;
    q.stages = (int)std::min<size_t>(PX_STAGES, budget / x_stage);
    q.W = B; q.ldw = ldb; q.out = Y; q.ldo = ldy; q.bias = bias;
    if (rb) { q.relu_src = rb->src; q.ld_relu = rb->ld; q.colsum = rb->colsum; }
    CUtensorMap tx, ty;
    RNN_TRY(make_map(&tx, A, Kred, M, lda, BK, BM));
    RNN_TRY(make_map(&ty, Y, N, M, ldy, 32, 32, false, /*swizzle=*/false));
    const int64_t per_n =
        std::max<int64_t>(1, std::min<int64_t>(num_sms() / q.n_tiles_n, q.n_tiles_m));
    const unsigned grid = (unsigned)(per_n * q.n_tiles_n);
    const size_t smem = q.stages * x_stage + 1024 + tscratch;
    auto kern = s3 ? tc_projt_kernel<PM_3X>
                : prec == RNN_PREC_BF16 ? tc_projt_kernel<PM_BF16> : tc_projt_kernel<PM_TF32>;
    RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, PT_THREADS, smem, st>>>(tx, ty, q);
    RNN_LAUNCH_CHECK();
    if (rb) { rb->fused = true; rb->grid = (int)grid; rb->n_tiles_n = q.n_tiles_n; }
    return RNN_OK;
  }
  {
    // persistent resident-B kernel when B's column block fits next to a 2-deep A ring
    const bool s3 = prec == RNN_PREC_3XTF32;
    const int nkb = (int)ceil_div(Kred, BK);
    const int n_tiles_n = (int)ceil_div(N, 128);
    const int BN = (int)((ceil_div(N, n_tiles_n) + 15) / 16 * 16);
    const size_t b_res = (size_t)BN * BK * 4 * nkb * (s3 ? 2 : 1);
    const size_t a_stage = (size_t)BM * BK * 4 * (s3 ? 2 : 1);
    const size_t budget = 227 * 1024 - 1024 - 256;
    if (b_res + 2 * a_stage <= budget && n_tiles_n <= num_sms()) {
      ProjParams q{};
      q.M = M; q.N = N; q.BN = BN; q.n_tiles_n = n_tiles_n;
      q.n_tiles_m = ceil_div(M, BM);
      q.nkb = nkb;
      q.stages = (int)std::min<size_t>(PT_MAX_STAGES, (budget - b_res) / a_stage);
      q.out = Y; q.ldo = ldy; q.bias = bias;
      q.tmem_cols = pow2_cols(2 * BN);
      CUtensorMap ta, tb;
      RNN_TRY(make_map(&ta, A, Kred, M, lda, BK, BM));
      RNN_TRY(make_map(&tb, B, Kred, N, ldb, BK, (uint32_t)BN));
      const int64_t per_n = std::max<int64_t>(1, std::min<int64_t>(num_sms() / n_tiles_n, q.n_tiles_m));
      const unsigned grid = (unsigned)(per_n * n_tiles_n);
      const size_t smem = b_res + q.stages * a_stage + 1024 + 8 * (3 * PT_MAX_STAGES + 6) + 64;
      auto kern = s3 ? tc_proj_kernel<PM_3X>
                  : prec == RNN_PREC_BF16 ? tc_proj_kernel<PM_BF16> : tc_proj_kernel<PM_TF32>;
      RNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<grid, PT_THREADS, smem, st>>>(ta, tb, q);
      RNN_LAUNCH_CHECK();
      return RNN_OK;
    }
  }
  GemmParams p{};
  p.M = M; p.N = N;
  p.BN = N <= 256 ? (int)((N + 15) / 16 * 16) : 256;
  p.Kred = Kred; p.k_split = ceil_div(Kred, BK) * BK;
  p.out = Y; p.ldo = ldy; p.bias = bias; p.mode = 0;
  const bool blo = b_has_lo && prec == RNN_PREC_3XTF32 && !getenv("RNN_NO_BLO");
  p.b_lo_row = blo ? N : 0;
  CUtensorMap ta, tb;
  RNN_TRY(make_map(&ta, A, Kred, M, lda, BK, BM));
  RNN_TRY(make_map(&tb, B, Kred, blo ? 2 * (int64_t)N : N, ldb, BK, (uint32_t)p.BN));
  return gemm<false, false>(ta, tb, p, 1, prec, st);
}

}  // namespace
}  // namespace rnn

using namespace rnn;

extern "C" rnn_status rnn_project(const float* X, int64_t M, int32_t K, int64_t ldx,
                                  const float* W, int32_t N, int64_t ldw, const float* bias,
                                  float* Y, int64_t ldy, rnn_precision prec, void* stream) {
  clear_error();
  RNN_REQUIRE(X && W && Y, RNN_ERR_INVALID_ARGUMENT, "X, W, Y required");
  RNN_REQUIRE(M >= 0 && M < (int64_t(1) << 31) && K >= 0 && K <= 8192 && N >= 1 && N <= 8192,
              RNN_ERR_UNSUPPORTED, "shape outside M < 2^31, K <= 8192, 1 <= N <= 8192");
  RNN_REQUIRE(ldx >= K && ldw >= K && ldy >= N, RNN_ERR_INVALID_ARGUMENT, "ld too small");
  RNN_REQUIRE(prec == RNN_PREC_TF32 || prec == RNN_PREC_3XTF32 || prec == RNN_PREC_BF16,
              RNN_ERR_INVALID_ARGUMENT,
              "precision");
  return gemm_kk(X, M, K, ldx, W, N, ldw, bias, Y, ldy, prec, as_stream(stream));
}

namespace {
struct BwdWs {
  float* Wt; float* dWt; float* part; float* part2; float* cpart; float* rpart;
  size_t bytes;
  int splits; int64_t chunks;
};
// dW for a wide dY (N > 128) and K <= 128 is computed transposed, dW^T = X^T dY: one 128-row
// MMA tile over k and N = 256 columns of n per MMA, so X is re-read ceil(N / 256) times instead
// of ceil(N / 128) and the shared-memory reads per loaded byte drop (the 3xTF32 tile GEMM is
// bound by shared-memory traffic); the ordered reduce writes dW^T, a small transpose gives dW.
#ifndef RNN_DW_MAX_CHAIN
#define RNN_DW_MAX_CHAIN 2048
#endif
constexpr int64_t DW_MAX_CHAIN = RNN_DW_MAX_CHAIN;
constexpr int64_t RELU_PART_ROWS = 1024;   // >= the fused kernel's grid (SMs, or column blocks)
inline bool dw_swapped(int K, int N) { return N > 128 && K <= 128 && !getenv("RNN_NO_DWT"); }

BwdWs bwd_ws(int64_t M, int K, int N, void* base) {
  BwdWs w{};
  Carve c(base);
  const int64_t ldt = (N + 3) / 4 * 4;
  w.Wt = c.take<float>((size_t)2 * K * ldt);   // W^T hi (rows 0..K-1) and lo (rows K..2K-1)
  w.dWt = c.take<float>((size_t)K * N);
  const int64_t tiles = dw_swapped(K, N) ? ceil_div(K, BM) * ceil_div(N, 256)
                                         : ceil_div(N, BM) * ceil_div(K, 256);
  int64_t splits = ceil_div(M, 8 * BK);
  const int64_t cap = (148 + tiles - 1) / tiles;   // about one wave of CTAs
  if (splits > cap) splits = cap;
  // Precision: the tensor core's fp32 accumulate rounds every partial sum, so the dW error
  // grows linearly with the rows one split accumulates (measured on B200, 3xTF32 max error
  // 1.35e-5 at 704 rows per split, 1.5e-4 at 6,757 -- profiles/r02/precision); bound the
  // chain at DW_MAX_CHAIN rows and leave the rest to the fixed-order fp32 split reduction
  // (a drain-to-registers variant kept the chain short inside one CTA but cost 48 % on the
  // wide MAG shapes -- profiles/r02/cmp).
  // (whole waves: a partial second wave of CTAs would cost a full wave's time)
  const int64_t min_splits = ceil_div(M, DW_MAX_CHAIN);
  if (splits < min_splits) splits = ceil_div(min_splits, cap) * cap;
  if (splits < 1) splits = 1;
  w.splits = (int)splits;
  w.part = c.take<float>((size_t)splits * N * K);
  w.part2 = c.take<float>((size_t)ceil_div(splits, 8) * N * K);
  w.chunks = ceil_div(M > 0 ? M : 1, 4096);
  w.cpart = c.take<float>((size_t)w.chunks * N);
  // ReLU-input column sums: one row per CTA of the fused kernel (<= RELU_PART_ROWS) or per
  // 4096-row chunk of the unfused path
  w.rpart = c.take<float>((size_t)std::max<int64_t>(RELU_PART_ROWS, w.chunks) * K);
  w.bytes = c.used + 1024;
  return w;
}
}  // namespace

extern "C" rnn_status rnn_project_bwd_workspace_size(int64_t M, int32_t K, int32_t N,
                                                     size_t* bytes) {
  clear_error();
  RNN_REQUIRE(bytes && M >= 0 && K >= 0 && N >= 1, RNN_ERR_INVALID_ARGUMENT, "bad argument");
  *bytes = bwd_ws(M, K, N, nullptr).bytes;
  return RNN_OK;
}

namespace {
rnn_status project_bwd(const float* X, int64_t M, int32_t K, int64_t ldx, const float* W, int32_t N,
                       int64_t ldw, const float* dY, int64_t lddy, float* dX, int64_t lddx,
                       float* dW, float* db, bool relu_in, float* d_in_bias, rnn_precision prec,
                       void* workspace, size_t workspace_bytes, void* stream) {
  RNN_REQUIRE(X && W && dY && dW, RNN_ERR_INVALID_ARGUMENT, "X, W, dY, dW required");
  RNN_REQUIRE(prec == RNN_PREC_TF32 || prec == RNN_PREC_3XTF32 || prec == RNN_PREC_BF16,
              RNN_ERR_INVALID_ARGUMENT, "precision");
  RNN_REQUIRE(M >= 0 && M < (int64_t(1) << 31) && K >= 1 && K <= 8192 && N >= 1 && N <= 8192,
              RNN_ERR_UNSUPPORTED, "shape outside M < 2^31, 1 <= K <= 8192, 1 <= N <= 8192");
  RNN_REQUIRE(ldx >= K && ldw >= K && lddy >= N && (!dX || lddx >= K), RNN_ERR_INVALID_ARGUMENT,
              "ld too small");
  cudaStream_t st = as_stream(stream);
  BwdWs w = bwd_ws(M, K, N, workspace);
  RNN_REQUIRE(workspace && workspace_bytes >= w.bytes, RNN_ERR_WORKSPACE_TOO_SMALL,
              "workspace %zu < %zu bytes", workspace_bytes, w.bytes);
  const int64_t ldt = (N + 3) / 4 * 4;
  // dX = dY W : K-major A = dY [M, N], K-major B = W^T [K, N]
  if (dX) {
    transpose_hilo_kernel<<<(unsigned)ceil_div((int64_t)N * K, 256), 256, 0, st>>>(W, N, K, ldw, w.Wt,
                                                                             ldt);
    RNN_LAUNCH_CHECK();
    ReluBwd rb{X, ldx, w.rpart, false, 0, 0};
    RNN_TRY(gemm_kk(dY, M, N, lddy, w.Wt, K, ldt, nullptr, dX, lddx, prec, st, true,
                    relu_in ? &rb : nullptr));
    if (relu_in && M > 0) {
      if (!rb.fused) {
        relu_mask_kernel<<<(unsigned)ceil_div(M * K, 256), 256, 0, st>>>(dX, lddx, X, ldx, M, K);
        RNN_LAUNCH_CHECK();
      }
      if (d_in_bias) {
        if (rb.fused) {
          RNN_REQUIRE(rb.grid <= RELU_PART_ROWS, RNN_ERR_UNSUPPORTED, "fused grid %d", rb.grid);
          projt_colsum_final<<<(unsigned)ceil_div(K, 32), 256, 0, st>>>(w.rpart, rb.grid,
                                                                        rb.n_tiles_n, K, d_in_bias);
        } else {
          dim3 g1((unsigned)ceil_div(K, 32), (unsigned)w.chunks);
          colsum_partial<<<g1, 256, 0, st>>>(dX, M, K, lddx, 4096, w.rpart);
          colsum_final<<<(unsigned)ceil_div(K, 32), 256, 0, st>>>(w.rpart, w.chunks, K,
                                                                   d_in_bias);
        }
        RNN_LAUNCH_CHECK();
      }
    } else if (relu_in && d_in_bias) {
      RNN_CUDA(cudaMemsetAsync(d_in_bias, 0, sizeof(float) * K, st));
    }
  }
  // dW = dY^T X : both operands MN-major, split over M, ordered reduction
  if (M == 0) {
    RNN_CUDA(cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)N * K, st));
  } else if (dw_swapped(K, N)) {
    // dW^T [K, N] = X^T dY: A = X (MN-major, M = k), B = dY (MN-major, N = n, 256 per tile)
    GemmParams p{};
    p.M = K; p.N = N;
    p.BN = N <= 256 ? (int)((N + 31) / 32 * 32) : 256;
    p.Kred = M;
    p.k_split = ceil_div(ceil_div(M, w.splits), BK) * BK;
    const int splits = (int)ceil_div(M, p.k_split);
    p.mode = 1; p.partial = w.part; p.ldp = N; p.part_stride = (int64_t)N * K;
    p.smem_kb = 100;   // 2 CTAs / SM: measured 1.40 -> 1.23 ms at N = 768 (profiles/r01/dw)
    CUtensorMap ta, tb;
    p.a3d = map3_ok(X, K, ldx);
    p.b3d = map3_ok(dY, N, lddy);
    if (p.a3d) RNN_TRY(make_map3(&ta, X, K, M, ldx, 16, BM / 32));
    else RNN_TRY(make_map(&ta, X, K, M, ldx, 32, 16, true));
    if (p.b3d) RNN_TRY(make_map3(&tb, dY, N, M, lddy, 16, (uint32_t)(p.BN / 32)));
    else RNN_TRY(make_map(&tb, dY, N, M, lddy, 32, 16, true));
    RNN_TRY((gemm<true, true>(ta, tb, p, splits, prec, st)));
    const int64_t nk = (int64_t)N * K;
    if (nk % 4 == 0) {
      const int64_t groups = ceil_div(splits, 8);
      splitk_stage<<<dim3((unsigned)ceil_div(nk / 4, 128), (unsigned)groups), 128, 0, st>>>(
          w.part, splits, p.part_stride, nk, w.part2);
      splitk_final<<<(unsigned)ceil_div(nk / 4, 128), 128, 0, st>>>(w.part2, groups, nk, w.dWt);
    } else
      splitk_reduce1<<<(unsigned)ceil_div(nk, 128), 128, 0, st>>>(w.part, splits, p.part_stride,
                                                                  nk, w.dWt);
    RNN_LAUNCH_CHECK();
    // dW [N, K] = (dW^T [K, N])^T
    transpose_kernel<<<(unsigned)ceil_div(nk, 256), 256, 0, st>>>(w.dWt, K, N, N, dW, K);
    RNN_LAUNCH_CHECK();
  } else {
    GemmParams p{};
    p.M = N; p.N = K;
    p.BN = K <= 256 ? (int)((K + 31) / 32 * 32) : 256;
    p.Kred = M;
    p.k_split = ceil_div(ceil_div(M, w.splits), BK) * BK;
    const int splits = (int)ceil_div(M, p.k_split);
    p.mode = 1; p.partial = w.part; p.ldp = K; p.part_stride = (int64_t)N * K;
    CUtensorMap ta, tb;
    p.a3d = map3_ok(dY, N, lddy);
    p.b3d = map3_ok(X, K, ldx);
    if (p.a3d) RNN_TRY(make_map3(&ta, dY, N, M, lddy, 16, BM / 32));
    else RNN_TRY(make_map(&ta, dY, N, M, lddy, 32, 16, true));
    if (p.b3d) RNN_TRY(make_map3(&tb, X, K, M, ldx, 16, (uint32_t)(p.BN / 32)));
    else RNN_TRY(make_map(&tb, X, K, M, ldx, 32, 16, true));
    RNN_TRY((gemm<true, true>(ta, tb, p, splits, prec, st)));
    // partial tiles and dW are contiguous [N, K]
    const int64_t nk = (int64_t)N * K;
    if (nk % 4 == 0 && aligned16(dW)) {
      const int64_t groups = ceil_div(splits, 8);
      splitk_stage<<<dim3((unsigned)ceil_div(nk / 4, 128), (unsigned)groups), 128, 0, st>>>(
          w.part, splits, p.part_stride, nk, w.part2);
      splitk_final<<<(unsigned)ceil_div(nk / 4, 128), 128, 0, st>>>(w.part2, groups, nk, dW);
    } else
      splitk_reduce1<<<(unsigned)ceil_div(nk, 128), 128, 0, st>>>(w.part, splits, p.part_stride,
                                                                  nk, dW);
    RNN_LAUNCH_CHECK();
  }
  if (db) {
    if (M == 0) {
      RNN_CUDA(cudaMemsetAsync(db, 0, sizeof(float) * N, st));
    } else {
      dim3 g1((unsigned)ceil_div(N, 32), (unsigned)w.chunks);
      colsum_partial<<<g1, 256, 0, st>>>(dY, M, N, lddy, 4096, w.cpart);
      colsum_final<<<(unsigned)ceil_div(N, 32), 256, 0, st>>>(w.cpart, w.chunks, N, db);
      RNN_LAUNCH_CHECK();
    }
  }
  return RNN_OK;
}
}  // namespace

extern "C" rnn_status rnn_project_bwd(const float* X, int64_t M, int32_t K, int64_t ldx,
                                      const float* W, int32_t N, int64_t ldw, const float* dY,
                                      int64_t lddy, float* dX, int64_t lddx, float* dW, float* db,
                                      rnn_precision prec, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  clear_error();
  return project_bwd(X, M, K, ldx, W, N, ldw, dY, lddy, dX, lddx, dW, db, false, nullptr, prec,
                     workspace, workspace_bytes, stream);
}

extern "C" rnn_status rnn_project_bwd_relu(const float* X, int64_t M, int32_t K, int64_t ldx,
                                           const float* W, int32_t N, int64_t ldw,
                                           const float* dY, int64_t lddy, float* dX, int64_t lddx,
                                           float* dW, float* db, float* d_in_bias,
                                           rnn_precision prec, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  clear_error();
  RNN_REQUIRE(dX, RNN_ERR_INVALID_ARGUMENT, "dX is required");
  return project_bwd(X, M, K, ldx, W, N, ldw, dY, lddy, dX, lddx, dW, db, true, d_in_bias, prec,
                     workspace, workspace_bytes, stream);
}

// Internal test hook (not part of include/rnn.h): C[M, N] = A . B with A given K-major
// ([M, Kred] row-major) or MN-major ([Kred, M] row-major), likewise B ([N, Kred] or [Kred, N]).
extern "C" rnn_status rnn_internal_gemm(int a_mn, int b_mn, const float* A, int64_t lda,
                                        const float* B, int64_t ldb, int64_t M, int N,
                                        int64_t Kred, float* Cout, int64_t ldc, int prec,
                                        void* stream) {
  clear_error();
  GemmParams p{};
  p.M = M; p.N = N;
  p.BN = N <= 256 ? (int)((N + 31) / 32 * 32) : 256;
  p.Kred = Kred; p.k_split = ceil_div(Kred, BK) * BK;
  p.out = Cout; p.ldo = ldc; p.mode = 0;
  CUtensorMap ta, tb;
  const uint32_t kb_rows = (a_mn && b_mn) ? 16 : BK;   // launch_gemm's stage depth (KB)
  if (a_mn) RNN_TRY(make_map(&ta, A, M, Kred, lda, 32, kb_rows, true));
  else RNN_TRY(make_map(&ta, A, Kred, M, lda, BK, BM));
  if (b_mn) RNN_TRY(make_map(&tb, B, N, Kred, ldb, 32, kb_rows, true));
  else RNN_TRY(make_map(&tb, B, Kred, N, ldb, BK, (uint32_t)p.BN));
  const rnn_precision pr = (rnn_precision)prec;
  cudaStream_t st = as_stream(stream);
  if (a_mn && b_mn) return gemm<true, true>(ta, tb, p, 1, pr, st);
  if (a_mn) return gemm<true, false>(ta, tb, p, 1, pr, st);
  if (b_mn) return gemm<false, true>(ta, tb, p, 1, pr, st);
  return gemm<false, false>(ta, tb, p, 1, pr, st);
}

extern "C" int rnn_internal_proj_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, rnn::g_proj_stats, sizeof(unsigned long long) * 16) != cudaSuccess)
    return 1;
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(rnn::g_proj_stats, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}

extern "C" int rnn_internal_gemm_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, rnn::g_gemm_stats, sizeof(unsigned long long) * 16) != cudaSuccess)
    return 1;
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(rnn::g_gemm_stats, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
