// join_index.cu -- A1: the join-index builder (replaces cuDF merge + groupby, PAPER.md:751,
// :755).  Built once per (E, S, T) and reused every iteration ("content caching").
//
// Pipeline (all on device, deterministic):
//   1. key -> row hash tables for S and T (open addressing, splitmix64 hash, 64-bit CAS;
//      a second insert of a key is a duplicate => RNN_ERR_DUPLICATE_KEY).
//   2. probe every E row (natural join: rows whose s or t has no partner are dropped,
//      PAPER.md:321-326); stable compaction by an exclusive scan of the hit flags.
//   3. group order: T keys are radix-sorted once to ranks; the join rows are stably radix
//      sorted by rank(t) (or by the raw signed key when T is absent, or by
//      (rank t, rank s) for the DHN adjacency variant).  Stability keeps edge-row order
//      inside a group.  Head flags + scan give group ids, group_ptr, group_key.
//   4. transposed CSR: counts per S row + scan -> src_ptr; stable radix sort of positions
//      by src_row -> src_pos; src_group = group of each position.
//   5. work schedules over both CSRs (see build_schedule).
#include <algorithm>

#include "common.cuh"

namespace rnn {
namespace {

constexpr int T256 = 256;
constexpr uint64_t EMPTY_KEY = 0x8000000000000000ull;  // INT64_MIN, kept in a side slot

inline unsigned blocks_for(int64_t n, int t = T256) {
  int64_t b = ceil_div(n > 0 ? n : 1, t);
  return (unsigned)(b > 2147483647 ? 2147483647 : b);
}

inline int64_t pow2_at_least(int64_t x) {
  int64_t c = 2;
  while (c < x) c <<= 1;
  return c;
}

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

struct Table {
  unsigned long long* keys;  // [cap] EMPTY_KEY = free
  int32_t* rows;             // [cap]
  int32_t* sentinel_row;     // row holding key INT64_MIN, or -1
  int64_t mask;
};

__global__ void table_init(Table t) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i <= t.mask) { t.keys[i] = EMPTY_KEY; t.rows[i] = -1; }
  if (i == 0) *t.sentinel_row = -1;
}

__global__ void table_insert(Table t, const int64_t* __restrict__ keys, int64_t n, int* dup) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = (unsigned long long)keys[i];
  if (k == EMPTY_KEY) {
    if (atomicCAS(t.sentinel_row, -1, (int32_t)i) != -1) atomicExch(dup, 1);
    return;
  }
  int64_t h = (int64_t)(splitmix64(k) & (uint64_t)t.mask);
  while (true) {
    unsigned long long prev = atomicCAS(&t.keys[h], EMPTY_KEY, k);
    if (prev == EMPTY_KEY) { t.rows[h] = (int32_t)i; return; }
    if (prev == k) { atomicExch(dup, 1); return; }
    h = (h + 1) & t.mask;
  }
}

__device__ __forceinline__ int32_t table_find(const Table& t, int64_t key) {
  const unsigned long long k = (unsigned long long)key;
  if (k == EMPTY_KEY) return *t.sentinel_row;
  int64_t h = (int64_t)(splitmix64(k) & (uint64_t)t.mask);
  while (true) {
    unsigned long long c = t.keys[h];
    if (c == k) return t.rows[h];
    if (c == EMPTY_KEY) return -1;
    h = (h + 1) & t.mask;
  }
}

// probe: s_row_of[j], t_row_of[j], hit[j] in {0,1} (as int64 for the scan)
__global__ void probe_kernel(const int64_t* __restrict__ e_src, const int64_t* __restrict__ e_dst,
                             int64_t n_e, Table S, bool has_s, Table T, bool has_t,
                             int32_t* s_row_of, int32_t* t_row_of, int64_t* hit,
                             const uint8_t* __restrict__ e_mask) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n_e) return;
  int32_t sr = -1, tr = -1;
  bool ok = !e_mask || e_mask[j];   // selection sigma(E) pushed into the probe
  if (ok && has_s) { sr = table_find(S, e_src[j]); ok = sr >= 0; }
  if (ok && has_t) { tr = table_find(T, e_dst[j]); ok = tr >= 0; }
  s_row_of[j] = sr;
  t_row_of[j] = tr;
  hit[j] = ok ? 1 : 0;
}

// flipped signed key: unsigned order == signed order
__device__ __forceinline__ uint64_t flip(int64_t k) { return (uint64_t)k ^ 0x8000000000000000ull; }

__global__ void fill_sort_input_keys(const int64_t* __restrict__ keys, int64_t n, uint64_t* k,
                                     int32_t* v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) { k[i] = flip(keys[i]); v[i] = (int32_t)i; }
}

__global__ void ranks_from_sorted(const int32_t* __restrict__ sorted_rows, int64_t n,
                                  uint32_t* rank) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) rank[sorted_rows[r]] = (uint32_t)r;
}

// compaction of the join rows + their sort keys.  mode 0: key = rank_t[t_row];
// mode 1: key = flip(e_dst); mode 2: key = rank_t[t_row] * n_s + rank_s[s_row]
__global__ void compact_kernel(const int64_t* __restrict__ hit_scan, int64_t n_e,
                               const int64_t* __restrict__ e_dst,
                               const int32_t* __restrict__ s_row_of,
                               const int32_t* __restrict__ t_row_of,
                               const uint32_t* __restrict__ rank_t,
                               const uint32_t* __restrict__ rank_s, int64_t n_s, int mode,
                               uint64_t* key, int32_t* val) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n_e) return;
  int64_t p = hit_scan[j];
  if (hit_scan[j + 1] == p) return;  // not a join row
  uint64_t k;
  if (mode == 0) k = rank_t[t_row_of[j]];
  else if (mode == 1) k = flip(e_dst[j]);
  else k = (uint64_t)rank_t[t_row_of[j]] * (uint64_t)n_s + rank_s[s_row_of[j]];
  key[p] = k;
  val[p] = (int32_t)j;
}

// head flags of the sorted rows (group starts).  mode 2 compares key / n_s.
__global__ void head_kernel(const uint64_t* __restrict__ key, int64_t n, int mode, int64_t n_s,
                            int64_t* head) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (p == 0) { head[p] = 1; return; }
  uint64_t a = key[p], b = key[p - 1];
  if (mode == 2) { a /= (uint64_t)n_s; b /= (uint64_t)n_s; }
  head[p] = a != b ? 1 : 0;
}

struct IndexOut {
  int64_t* group_ptr; int64_t* group_key; int32_t* group_dst_row;
  int32_t* src_row; int32_t* edge_row;
};

__global__ void emit_groups(const int64_t* __restrict__ head_scan /*exclusive, [n+1]*/, int64_t n,
                            const int32_t* __restrict__ sorted_j, const int64_t* __restrict__ e_dst,
                            const int32_t* __restrict__ s_row_of,
                            const int32_t* __restrict__ t_row_of, IndexOut o, int32_t* pos_group) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t j = sorted_j[p];
  const int64_t h0 = head_scan[p];
  const bool is_head = head_scan[p + 1] != h0;
  const int64_t g = is_head ? h0 : h0 - 1;
  if (is_head) {
    o.group_ptr[g] = p;
    o.group_key[g] = e_dst[j];
    o.group_dst_row[g] = t_row_of[j];
  }
  if (p == n - 1) o.group_ptr[head_scan[n]] = n;
  o.src_row[p] = s_row_of[j];
  o.edge_row[p] = j;
  if (pos_group) pos_group[p] = (int32_t)g;
}

// dense groups (RNN_IDX_DENSE_GROUPS): group = rank of the T key; count group sizes
__global__ void emit_dense(const uint32_t* __restrict__ rank_t, int64_t n,
                           const int32_t* __restrict__ sorted_j,
                           const int32_t* __restrict__ s_row_of,
                           const int32_t* __restrict__ t_row_of, IndexOut o, int32_t* pos_group) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t j = sorted_j[p];
  const int64_t g = rank_t[t_row_of[j]];
  o.src_row[p] = s_row_of[j];
  o.edge_row[p] = j;
  pos_group[p] = (int32_t)g;
  atomicAdd(reinterpret_cast<unsigned long long*>(&o.group_ptr[g]), 1ull);
}

__global__ void dense_groups(const uint32_t* __restrict__ rank_t, int64_t n_t,
                             const int64_t* __restrict__ dst_key, int64_t* group_key,
                             int32_t* group_dst_row) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_t) return;
  const uint32_t g = rank_t[i];
  group_key[g] = dst_key[i];
  group_dst_row[g] = (int32_t)i;
}

__global__ void count_src(const int32_t* __restrict__ src_row, int64_t n, int64_t* cnt) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[src_row[p]]), 1ull);
}

__global__ void transpose_input(const int32_t* __restrict__ src_row, int64_t n, uint32_t* k,
                                int32_t* v) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) { k[p] = (uint32_t)src_row[p]; v[p] = (int32_t)p; }
}

__global__ void src_group_kernel(const int32_t* __restrict__ src_pos, int64_t n,
                                 const int32_t* __restrict__ pos_group,
                                 const uint32_t* __restrict__ sorted_src, int32_t* src_group,
                                 int32_t* src_seg) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) {
    src_group[q] = pos_group[src_pos[q]];
    src_seg[q] = (int32_t)sorted_src[q];
  }
}

// ------------------------------------------------------------------------------------------
// work schedule over a CSR ptr[n_seg+1] with E = ptr[n_seg] positions.
// Candidate boundaries (positions), then sort + unique:
//   (a) for every C-block b: the end of the segment containing position b*C (or b*C itself
//       when a segment starts exactly there), kept only if it lies inside block b;
//   (b) for every segment longer than C: its start, its end and the interior boundaries of
//       ceil(len/C) near-equal pieces;
//   (c) 0 and E.
// Small segments are never split; every long segment's start and end are boundaries, so
// its pieces are exactly the consecutive items [lower_bound(start), lower_bound(end)).
// ------------------------------------------------------------------------------------------
__global__ void sched_block_candidates(const int64_t* __restrict__ ptr, int64_t n_seg, int64_t E,
                                       int64_t C, int64_t n_blocks, uint64_t* cand) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  const int64_t x = b * C;
  int64_t out = E;  // E is always a boundary, so a duplicate of it is harmless
  // segment containing x: last s with ptr[s] <= x (skip empties: they share the start)
  int64_t s = upper_bound_dev(ptr, 0, n_seg + 1, x) - 1;
  if (s >= 0 && s < n_seg) {
    if (ptr[s] == x) out = x;
    else {
      int64_t end = ptr[s + 1];
      out = end < x + C ? end : E;
    }
  }
  cand[b] = (uint64_t)out;
}

__global__ void sched_long_counts(const int64_t* __restrict__ ptr, int64_t n_seg, int64_t C,
                                  int64_t* cnt) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  int64_t len = ptr[s + 1] - ptr[s];
  cnt[s] = len > C ? ceil_div_dev(len, C) + 1 : 0;  // pieces + 1 boundaries (start .. end)
}

__global__ void sched_long_emit(const int64_t* __restrict__ ptr, int64_t n_seg, int64_t C,
                                const int64_t* __restrict__ off, uint64_t* cand) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  int64_t a = ptr[s], len = ptr[s + 1] - a;
  if (len <= C) return;
  int64_t k = (len + C - 1) / C;
  uint64_t* o = cand + off[s];
  for (int64_t i = 0; i <= k; ++i) o[i] = (uint64_t)(a + (len * i) / k);
}

__global__ void unique_heads(const uint64_t* __restrict__ v, int64_t n, int64_t* head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || v[i] != v[i - 1]) ? 1 : 0;
}

__global__ void unique_emit(const uint64_t* __restrict__ v, int64_t n,
                            const int64_t* __restrict__ hs, int64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && hs[i + 1] != hs[i]) out[hs[i]] = (int64_t)v[i];
}


struct Sched {
  // device scratch sizes for one schedule build
  static size_t bytes(int64_t n_seg, int64_t E, int64_t C) {
    const int64_t n_blocks = ceil_div(E > 0 ? E : 1, C);
    size_t b = 0;
    auto add = [&](size_t x) { b = ((b + 255) & ~size_t(255)) + x; };
    const int64_t cap = n_blocks + 2 + 2 * ceil_div(E > 0 ? E : 1, C) + E / (C + 1) + 2;
    add(sizeof(int64_t) * (n_seg + 1));     // long counts / offsets
    add(scan_workspace_bytes(std::max<int64_t>(n_seg, cap)));
    add(sizeof(uint64_t) * cap);            // candidates
    add(sizeof(int32_t) * cap);             // dummy values for the sort
    add(sizeof(int64_t) * (cap + 1));       // unique heads
    add(radix_sort_workspace_bytes(cap));
    return b + 256;
  }
};

// first segment an item touches: the segment holding position work_ptr[i] (or, when empty
// segments start exactly there, the first of them)
__global__ void sched_seg_kernel(const int64_t* __restrict__ ptr, int64_t n_seg,
                                 const int64_t* __restrict__ wp, int64_t n_items, int32_t* seg) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const int64_t b = wp[i];
  int64_t s = lower_bound_dev(ptr, 0, n_seg + 1, b);
  if (s > n_seg || ptr[s] > b) s -= 1;
  seg[i] = (int32_t)s;
}

// host: returns the number of items; writes work_ptr[n+1] (and work_seg[n]) when out != nullptr.
rnn_status build_schedule(const int64_t* ptr, int64_t n_seg, int64_t E, int64_t C, void* ws,
                          int64_t* out, int32_t* seg_out, int64_t* n_items, cudaStream_t st) {
  if (E <= 0) {
    *n_items = 0;
    if (out) RNN_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    return RNN_OK;
  }
  const int64_t n_blocks = ceil_div(E, C);
  Carve c(ws);
  // long-segment boundary counts: sum over long segs of (ceil(len/C)+1) <= 2E/C + ... bound
  const int64_t cap = n_blocks + 2 + 2 * ceil_div(E, C) + E / (C + 1) + 2;
  int64_t* cnt = c.take<int64_t>(n_seg + 1);
  void* sws = c.take<char>(scan_workspace_bytes(std::max<int64_t>(n_seg, cap)));
  uint64_t* cand = c.take<uint64_t>(cap);
  int32_t* dummy = c.take<int32_t>(cap);
  int64_t* head = c.take<int64_t>(cap + 1);
  void* rws = c.take<char>(radix_sort_workspace_bytes(cap));

  sched_block_candidates<<<blocks_for(n_blocks), T256, 0, st>>>(ptr, n_seg, E, C, n_blocks, cand);
  RNN_LAUNCH_CHECK();
  int64_t n_long_b = 0;
  if (n_seg > 0) {
    sched_long_counts<<<blocks_for(n_seg), T256, 0, st>>>(ptr, n_seg, C, cnt);
    RNN_LAUNCH_CHECK();
    RNN_TRY(exclusive_scan_i64(cnt, cnt, n_seg, sws, st));
    RNN_CUDA(cudaMemcpyAsync(&n_long_b, cnt + n_seg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RNN_CUDA(cudaStreamSynchronize(st));
    if (n_blocks + 2 + n_long_b > cap)
      RNN_FAIL(RNN_ERR_CUDA, "internal: schedule candidate overflow");
    sched_long_emit<<<blocks_for(n_seg), T256, 0, st>>>(ptr, n_seg, C, cnt, cand + n_blocks);
    RNN_LAUNCH_CHECK();
  }
  const uint64_t ends[2] = {0ull, (uint64_t)E};
  RNN_CUDA(cudaMemcpyAsync(cand + n_blocks + n_long_b, ends, sizeof(ends), cudaMemcpyHostToDevice, st));
  const int64_t n_cand = n_blocks + n_long_b + 2;
  RNN_CUDA(cudaMemsetAsync(dummy, 0, sizeof(int32_t) * n_cand, st));
  RNN_TRY(radix_sort_u64(cand, dummy, n_cand, bits_for((uint64_t)E), rws, st));
  unique_heads<<<blocks_for(n_cand), T256, 0, st>>>(cand, n_cand, head);
  RNN_LAUNCH_CHECK();
  RNN_TRY(exclusive_scan_i64(head, head, n_cand, sws, st));
  int64_t n_unique = 0;
  RNN_CUDA(cudaMemcpyAsync(&n_unique, head + n_cand, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RNN_CUDA(cudaStreamSynchronize(st));
  *n_items = n_unique - 1;  // boundaries include 0 and E
  if (out) {
    unique_emit<<<blocks_for(n_cand), T256, 0, st>>>(cand, n_cand, head, out);
    RNN_LAUNCH_CHECK();
    if (seg_out && *n_items > 0) {
      sched_seg_kernel<<<blocks_for(*n_items), T256, 0, st>>>(ptr, n_seg, out, *n_items, seg_out);
      RNN_LAUNCH_CHECK();
    }
  }
  return RNN_OK;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// entry point
// ------------------------------------------------------------------------------------------
namespace {

struct Plan {
  int64_t n_e, n_s, n_t, cap_s, cap_t, C;
  bool has_s, has_t, transpose, by_key;
};

size_t plan_bytes(const Plan& P) {
  size_t b = 0;
  auto add = [&](size_t x) { b = ((b + 255) & ~size_t(255)) + x; };
  const int64_t n = P.n_e > 0 ? P.n_e : 1;
  add(sizeof(unsigned long long) * P.cap_s); add(sizeof(int32_t) * P.cap_s); add(sizeof(int32_t));
  add(sizeof(unsigned long long) * P.cap_t); add(sizeof(int32_t) * P.cap_t); add(sizeof(int32_t));
  add(sizeof(int)); // dup flag
  add(sizeof(int32_t) * n); add(sizeof(int32_t) * n);      // s_row_of, t_row_of
  add(sizeof(int64_t) * (n + 1));                           // hit / scan
  add(sizeof(uint64_t) * n); add(sizeof(int32_t) * n);      // sort key / val
  add(sizeof(int64_t) * (n + 1));                           // head scan
  add(sizeof(int32_t) * n);                                 // pos_group
  add(sizeof(int64_t) * (P.n_t + 1));                       // dense group_ptr (phase 1)
  add(sizeof(uint32_t) * (P.n_t + 1)); add(sizeof(uint32_t) * (P.n_s + 1));  // ranks
  int64_t big = std::max<int64_t>(n, std::max(P.n_s, P.n_t));
  add(sizeof(uint64_t) * big); add(sizeof(int32_t) * big);  // rank sort scratch
  add(radix_sort_workspace_bytes(big));
  add(scan_workspace_bytes(big + 1));
  add(sizeof(int64_t) * (P.n_s + 2));                       // src counts
  add(std::max(Sched::bytes(n, n, P.C), Sched::bytes(P.n_s + 1, n, P.C)));
  return b + 1024;
}

struct Scratch {
  Table S, T;
  int* dup;
  int32_t *s_row_of, *t_row_of;
  int64_t* hit;
  uint64_t* key; int32_t* val;
  int64_t* head;
  int32_t* pos_group;
  int64_t* gp_dense;
  uint32_t *rank_t, *rank_s;
  uint64_t* rk; int32_t* rv;
  void* rsort_ws; void* scan_ws;
  int64_t* src_cnt;
  void* sched_ws;
};

Scratch carve(const Plan& P, void* ws) {
  Scratch s{};
  Carve c(ws);
  const int64_t n = P.n_e > 0 ? P.n_e : 1;
  s.S.keys = c.take<unsigned long long>(P.cap_s); s.S.rows = c.take<int32_t>(P.cap_s);
  s.S.sentinel_row = c.take<int32_t>(1); s.S.mask = P.cap_s - 1;
  s.T.keys = c.take<unsigned long long>(P.cap_t); s.T.rows = c.take<int32_t>(P.cap_t);
  s.T.sentinel_row = c.take<int32_t>(1); s.T.mask = P.cap_t - 1;
  s.dup = c.take<int>(1);
  s.s_row_of = c.take<int32_t>(n); s.t_row_of = c.take<int32_t>(n);
  s.hit = c.take<int64_t>(n + 1);
  s.key = c.take<uint64_t>(n); s.val = c.take<int32_t>(n);
  s.head = c.take<int64_t>(n + 1);
  s.pos_group = c.take<int32_t>(n);
  s.gp_dense = c.take<int64_t>(P.n_t + 1);
  s.rank_t = c.take<uint32_t>(P.n_t + 1); s.rank_s = c.take<uint32_t>(P.n_s + 1);
  int64_t big = std::max<int64_t>(n, std::max(P.n_s, P.n_t));
  s.rk = c.take<uint64_t>(big); s.rv = c.take<int32_t>(big);
  s.rsort_ws = c.take<char>(radix_sort_workspace_bytes(big));
  s.scan_ws = c.take<char>(scan_workspace_bytes(big + 1));
  s.src_cnt = c.take<int64_t>(P.n_s + 2);
  s.sched_ws = c.take<char>(std::max(Sched::bytes(n, n, P.C), Sched::bytes(P.n_s + 1, n, P.C)));
  return s;
}

rnn_status rank_keys(const int64_t* keys, int64_t n, Scratch& s, uint32_t* rank, cudaStream_t st) {
  if (n <= 0) return RNN_OK;
  fill_sort_input_keys<<<blocks_for(n), T256, 0, st>>>(keys, n, s.rk, s.rv);
  RNN_LAUNCH_CHECK();
  RNN_TRY(radix_sort_u64(s.rk, s.rv, n, 64, s.rsort_ws, st));
  ranks_from_sorted<<<blocks_for(n), T256, 0, st>>>(s.rv, n, rank);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

}  // namespace
}  // namespace rnn

using namespace rnn;

static rnn_status build_impl(const int64_t* e_src_key, const int64_t* e_dst_key,
                             int64_t n_edge_rows, const int64_t* src_key, int64_t n_src,
                             const int64_t* dst_key, int64_t n_dst, int flags,
                             int64_t rows_per_item, rnn_join_index* idx, void* workspace,
                             size_t* workspace_bytes, void* stream, const uint8_t* e_mask);

extern "C" rnn_status rnn_build_join_index(const int64_t* e_src_key, const int64_t* e_dst_key,
                                           int64_t n_edge_rows, const int64_t* src_key,
                                           int64_t n_src, const int64_t* dst_key, int64_t n_dst,
                                           int flags, int64_t rows_per_item, rnn_join_index* idx,
                                           void* workspace, size_t* workspace_bytes,
                                           void* stream) {
  clear_error();
  return build_impl(e_src_key, e_dst_key, n_edge_rows, src_key, n_src, dst_key, n_dst, flags,
                    rows_per_item, idx, workspace, workspace_bytes, stream, nullptr);
}

extern "C" rnn_status rnn_build_join_index_sel(const int64_t* e_src_key, const int64_t* e_dst_key,
                                               const uint8_t* e_mask, int64_t n_edge_rows,
                                               const int64_t* src_key, int64_t n_src,
                                               const int64_t* dst_key, int64_t n_dst, int flags,
                                               int64_t rows_per_item, rnn_join_index* idx,
                                               void* workspace, size_t* workspace_bytes,
                                               void* stream) {
  clear_error();
  RNN_REQUIRE(e_mask || n_edge_rows == 0, RNN_ERR_INVALID_ARGUMENT, "e_mask is NULL");
  return build_impl(e_src_key, e_dst_key, n_edge_rows, src_key, n_src, dst_key, n_dst, flags,
                    rows_per_item, idx, workspace, workspace_bytes, stream, e_mask);
}

namespace rnn {
namespace {
__global__ void select_kernel(const void* __restrict__ attr, int dtype, int64_t n, int op,
                              double value, int combine, uint8_t* __restrict__ mask) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  bool r;
  if (dtype == 0) {
    const int64_t a = static_cast<const int64_t*>(attr)[j];
    const int64_t v = (int64_t)value;
    r = op == 0 ? a == v : op == 1 ? a != v : op == 2 ? a < v : op == 3 ? a <= v
      : op == 4 ? a > v : a >= v;
  } else {
    const float a = static_cast<const float*>(attr)[j];
    const float v = (float)value;
    r = op == 0 ? a == v : op == 1 ? a != v : op == 2 ? a < v : op == 3 ? a <= v
      : op == 4 ? a > v : a >= v;
  }
  mask[j] = combine == 0 ? (uint8_t)r : combine == 1 ? (uint8_t)(mask[j] && r)
                                                      : (uint8_t)(mask[j] || r);
}
}  // namespace
}  // namespace rnn

extern "C" rnn_status rnn_select_mask(const void* attr, int32_t dtype, int64_t n, int32_t op,
                                      double value, int32_t combine, uint8_t* mask, void* stream) {
  clear_error();
  RNN_REQUIRE(n >= 0 && (n == 0 || (attr && mask)), RNN_ERR_INVALID_ARGUMENT, "bad argument");
  RNN_REQUIRE(dtype == 0 || dtype == 1, RNN_ERR_UNSUPPORTED, "dtype: 0 int64, 1 float32");
  RNN_REQUIRE(op >= 0 && op <= 5, RNN_ERR_INVALID_ARGUMENT, "op: EQ NE LT LE GT GE = 0..5");
  RNN_REQUIRE(combine >= 0 && combine <= 2, RNN_ERR_INVALID_ARGUMENT, "combine: 0 set, 1 and, 2 or");
  if (n == 0) return RNN_OK;
  select_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(attr, dtype, n, op,
                                                                          value, combine, mask);
  RNN_LAUNCH_CHECK();
  return RNN_OK;
}

static rnn_status build_impl(const int64_t* e_src_key, const int64_t* e_dst_key,
                             int64_t n_edge_rows, const int64_t* src_key, int64_t n_src,
                             const int64_t* dst_key, int64_t n_dst, int flags,
                             int64_t rows_per_item, rnn_join_index* idx, void* workspace,
                             size_t* workspace_bytes, void* stream, const uint8_t* e_mask) {
  RNN_REQUIRE(idx && workspace_bytes, RNN_ERR_INVALID_ARGUMENT, "idx and workspace_bytes required");
  RNN_REQUIRE(n_edge_rows >= 0 && n_src >= 0 && n_dst >= 0, RNN_ERR_INVALID_ARGUMENT,
              "negative size");
  RNN_REQUIRE(n_edge_rows == 0 || e_dst_key, RNN_ERR_INVALID_ARGUMENT, "e_dst_key is NULL");
  RNN_REQUIRE(!src_key || n_edge_rows == 0 || e_src_key, RNN_ERR_INVALID_ARGUMENT,
              "S given but e_src_key is NULL");
  RNN_REQUIRE(n_edge_rows < (int64_t(1) << 31) && n_src < (int64_t(1) << 31) &&
                  n_dst < (int64_t(1) << 31),
              RNN_ERR_UNSUPPORTED, "relations must have < 2^31 rows");
  const bool by_key = flags & RNN_IDX_WITHIN_GROUP_BY_SRC_KEY;
  const bool dense = flags & RNN_IDX_DENSE_GROUPS;
  RNN_REQUIRE(!dense || dst_key, RNN_ERR_INVALID_ARGUMENT, "RNN_IDX_DENSE_GROUPS needs T");
  RNN_REQUIRE(!by_key || (src_key && dst_key), RNN_ERR_UNSUPPORTED,
              "RNN_IDX_WITHIN_GROUP_BY_SRC_KEY needs S and T");
  RNN_REQUIRE(rows_per_item >= 0, RNN_ERR_INVALID_ARGUMENT, "rows_per_item < 0");
  Plan P{};
  P.n_e = n_edge_rows; P.n_s = src_key ? n_src : 0; P.n_t = dst_key ? n_dst : 0;
  P.has_s = src_key != nullptr; P.has_t = dst_key != nullptr;
  P.cap_s = pow2_at_least(2 * P.n_s + 2); P.cap_t = pow2_at_least(2 * P.n_t + 2);
  // default work-item size: 128 rows, smaller for small relations so that the schedule
  // still gives every SM several warps of work (Cora: 13k join rows -> 16-row items)
  if (rows_per_item > 0) {
    P.C = rows_per_item;
  } else {
    const int64_t per_warp = n_edge_rows / ((int64_t)num_sms() * 32);
    P.C = per_warp >= 128 ? 128 : per_warp <= 16 ? 16 : (per_warp + 15) / 16 * 16;
  }
  P.transpose = P.has_s && !(flags & RNN_IDX_NO_TRANSPOSE);
  P.by_key = by_key;
  if (by_key)
    RNN_REQUIRE((uint64_t)P.n_t * (uint64_t)(P.n_s > 0 ? P.n_s : 1) < (1ull << 63),
                RNN_ERR_UNSUPPORTED, "n_dst * n_src too large for the composite sort key");
  const size_t need = plan_bytes(P);
  const bool phase1 = idx->group_ptr == nullptr;
  if (!workspace) { *workspace_bytes = need; return RNN_OK; }
  RNN_REQUIRE(*workspace_bytes >= need, RNN_ERR_WORKSPACE_TOO_SMALL,
              "workspace %zu < %zu bytes", *workspace_bytes, need);
  cudaStream_t st = as_stream(stream);
  Scratch s = carve(P, workspace);
  const int64_t n_e = P.n_e;

  // 1. hash tables
  RNN_CUDA(cudaMemsetAsync(s.dup, 0, sizeof(int), st));
  table_init<<<blocks_for(P.cap_s), T256, 0, st>>>(s.S);
  table_init<<<blocks_for(P.cap_t), T256, 0, st>>>(s.T);
  RNN_LAUNCH_CHECK();
  if (P.has_s && P.n_s > 0) table_insert<<<blocks_for(P.n_s), T256, 0, st>>>(s.S, src_key, P.n_s, s.dup);
  if (P.has_t && P.n_t > 0) table_insert<<<blocks_for(P.n_t), T256, 0, st>>>(s.T, dst_key, P.n_t, s.dup);
  RNN_LAUNCH_CHECK();
  if (phase1 || (flags & RNN_IDX_VALIDATE)) {
    int dup = 0;
    RNN_CUDA(cudaMemcpyAsync(&dup, s.dup, sizeof(int), cudaMemcpyDeviceToHost, st));
    RNN_CUDA(cudaStreamSynchronize(st));
    RNN_REQUIRE(!dup, RNN_ERR_DUPLICATE_KEY, "S or T holds a repeated key (relations are sets)");
  }
  // 2. probe + compaction
  if (n_e > 0) {
    probe_kernel<<<blocks_for(n_e), T256, 0, st>>>(e_src_key, e_dst_key, n_e, s.S, P.has_s, s.T,
                                                   P.has_t, s.s_row_of, s.t_row_of, s.hit, e_mask);
    RNN_LAUNCH_CHECK();
  }
  RNN_TRY(exclusive_scan_i64(s.hit, s.hit, n_e, s.scan_ws, st));
  int64_t n_join = 0;
  RNN_CUDA(cudaMemcpyAsync(&n_join, s.hit + n_e, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RNN_CUDA(cudaStreamSynchronize(st));
  // 3. group order
  int mode = P.has_t ? (by_key ? 2 : 0) : 1;
  int bits = 64;
  if (P.has_t) RNN_TRY(rank_keys(dst_key, P.n_t, s, s.rank_t, st));
  if (by_key) RNN_TRY(rank_keys(src_key, P.n_s, s, s.rank_s, st));
  if (mode == 0) bits = bits_for((uint64_t)(P.n_t > 0 ? P.n_t - 1 : 0));
  if (mode == 2) bits = bits_for((uint64_t)P.n_t * (uint64_t)P.n_s);
  if (n_e > 0) {
    compact_kernel<<<blocks_for(n_e), T256, 0, st>>>(s.hit, n_e, e_dst_key, s.s_row_of,
                                                     s.t_row_of, s.rank_t, s.rank_s, P.n_s, mode,
                                                     s.key, s.val);
    RNN_LAUNCH_CHECK();
  }
  RNN_TRY(radix_sort_u64(s.key, s.val, n_join, bits, s.rsort_ws, st));
  if (n_join > 0) {
    head_kernel<<<blocks_for(n_join), T256, 0, st>>>(s.key, n_join, mode, P.n_s, s.head);
    RNN_LAUNCH_CHECK();
  }
  RNN_TRY(exclusive_scan_i64(s.head, s.head, n_join, s.scan_ws, st));
  int64_t n_groups = 0;
  RNN_CUDA(cudaMemcpyAsync(&n_groups, s.head + n_join, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RNN_CUDA(cudaStreamSynchronize(st));
  if (dense) n_groups = P.n_t;  // every T row is a group (key order), empty ones included

  idx->n_edge_rows = n_e; idx->n_join_rows = n_join; idx->n_groups = n_groups;
  idx->n_src_rows = P.n_s; idx->n_dst_rows = P.n_t;

  int64_t* out_gp; int64_t* out_gk; int32_t* out_gd; int32_t* out_sr; int32_t* out_er;
  if (phase1) {
    out_gp = s.hit;                                    // [n_join+1] <= [n_e+1]
    out_gk = reinterpret_cast<int64_t*>(s.rk);          // [G] <= big
    out_gd = s.rv;                                      // [G]
    out_sr = reinterpret_cast<int32_t*>(s.key);         // key (u64[n]) is free after head scan
    out_er = reinterpret_cast<int32_t*>(s.key) + (n_e > 0 ? n_e : 1);
  } else {
    RNN_REQUIRE(idx->group_key && idx->group_dst_row && idx->src_row && idx->edge_row &&
                    idx->pos_group && idx->work_ptr && idx->work_seg,
                RNN_ERR_INVALID_ARGUMENT, "phase 2 needs every group-major array");
    RNN_REQUIRE(!P.transpose || (idx->src_ptr && idx->src_pos && idx->src_group &&
                                 idx->src_seg && idx->src_work_ptr && idx->src_work_seg),
                RNN_ERR_INVALID_ARGUMENT, "phase 2 needs the transposed arrays");
    out_gp = idx->group_ptr; out_gk = idx->group_key; out_gd = idx->group_dst_row;
    out_sr = idx->src_row; out_er = idx->edge_row;
  }
  // sorted edge rows are in s.val; the emit kernel reads them before out_sr/out_er (which may
  // alias s.key in phase 1) are written -- s.val and s.key are distinct buffers.
  int32_t* pos_group = phase1 ? s.pos_group : idx->pos_group;
  if (dense) {
    // groups = all T rows in key order; sizes counted (exact integers), then scanned
    if (phase1) out_gp = s.gp_dense;
    RNN_CUDA(cudaMemsetAsync(out_gp, 0, sizeof(int64_t) * (P.n_t + 1), st));
    IndexOut o{out_gp, out_gk, out_gd, out_sr, out_er};
    if (n_join > 0) {
      emit_dense<<<blocks_for(n_join), T256, 0, st>>>(s.rank_t, n_join, s.val, s.s_row_of,
                                                      s.t_row_of, o, pos_group);
      RNN_LAUNCH_CHECK();
    }
    if (P.n_t > 0) {
      dense_groups<<<blocks_for(P.n_t), T256, 0, st>>>(s.rank_t, P.n_t, dst_key, out_gk, out_gd);
      RNN_LAUNCH_CHECK();
    }
    RNN_TRY(exclusive_scan_i64(out_gp, out_gp, P.n_t, s.scan_ws, st));
  } else if (n_join > 0) {
    IndexOut o{out_gp, out_gk, out_gd, out_sr, out_er};
    emit_groups<<<blocks_for(n_join), T256, 0, st>>>(s.head, n_join, s.val, e_dst_key,
                                                     s.s_row_of, s.t_row_of, o, pos_group);
    RNN_LAUNCH_CHECK();
  } else {
    RNN_CUDA(cudaMemsetAsync(out_gp, 0, sizeof(int64_t), st));
  }
  // 4. transposed CSR
  int64_t* out_sp = nullptr;
  if (P.transpose) {
    out_sp = phase1 ? s.src_cnt : idx->src_ptr;
    RNN_CUDA(cudaMemsetAsync(out_sp, 0, sizeof(int64_t) * (P.n_s + 1), st));
    if (n_join > 0) {
      count_src<<<blocks_for(n_join), T256, 0, st>>>(out_sr, n_join, out_sp);
      RNN_LAUNCH_CHECK();
    }
    RNN_TRY(exclusive_scan_i64(out_sp, out_sp, P.n_s, s.scan_ws, st));
    if (!phase1 && n_join > 0) {
      uint32_t* tk = reinterpret_cast<uint32_t*>(s.key);  // free now (phase 2)
      transpose_input<<<blocks_for(n_join), T256, 0, st>>>(out_sr, n_join, tk, idx->src_pos);
      RNN_LAUNCH_CHECK();
      RNN_TRY(radix_sort_u32(tk, idx->src_pos, n_join,
                             bits_for((uint64_t)(P.n_s > 0 ? P.n_s - 1 : 0)), s.rsort_ws, st));
      src_group_kernel<<<blocks_for(n_join), T256, 0, st>>>(idx->src_pos, n_join, pos_group, tk,
                                                            idx->src_group, idx->src_seg);
      RNN_LAUNCH_CHECK();
    }
  }
  // 5. schedules
  int64_t n_work = 0, n_src_work = 0;
  RNN_TRY(build_schedule(out_gp, n_groups, n_join, P.C, s.sched_ws,
                         phase1 ? nullptr : idx->work_ptr, phase1 ? nullptr : idx->work_seg,
                         &n_work, st));
  if (P.transpose)
    RNN_TRY(build_schedule(out_sp, P.n_s, n_join, P.C, s.sched_ws,
                           phase1 ? nullptr : idx->src_work_ptr,
                           phase1 ? nullptr : idx->src_work_seg, &n_src_work, st));
  idx->n_work = n_work;
  idx->n_src_work = P.transpose ? n_src_work : 0;
  if (!phase1) RNN_CUDA(cudaStreamSynchronize(st));
  return RNN_OK;
}
