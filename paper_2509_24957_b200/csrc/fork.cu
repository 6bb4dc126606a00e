// K3: copy-on-write branch-out on a paged KV block table, plus the
// difficulty-ordering segmented sort.
//
// The reference forks a branch by pure accounting: the child resumes the
// next template at the parent's position without re-charging the prefix
// (orchestrator.py:254-268 _spawn(offset_base=source.position), :384; the
// paper relies on vLLM prefix caching). On a paged KV cache
// that prefix reuse is a block-table duplication: the child shares the
// parent's full blocks (refcount += 1) and gets a private copy of the partial
// tail block. Allocation is an exclusive scan over tail-needing forks in
// (request, action) order, so tables, refcounts and the free cursor are
// bit-identical to the serial restatement (oracle/cow.py) regardless of
// scheduling. Chains (a child forked from a child of the same round) arrive
// pre-resolved to the table root by duchess_decide, and the root's rows are
// never written here, so forks are independent and run one CTA each.
#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kPlanWarps = 16;          // groups per plan CTA (one warp each)
constexpr int kScanThreads = 512;

__device__ __forceinline__ int group_count(const int32_t* counts, int stride, int g, int cap) {
  return counts ? min(max(counts[int64_t(g) * stride], 0), cap) : cap;
}

// Workspace (int32, zeroed before first use, self-cleaning afterwards):
//   gcount[G], gtail[G], tbase[G], rank[G * cap], meta[4] = {cursor, tails, done, -}
struct ForkWs {
  int32_t* gcount;
  int32_t* gtail;
  int32_t* tbase;
  int32_t* rank;
  int32_t* meta;
};

// Plan, one warp per group: each record's tail flag (prefix not on a block
// boundary) and its rank among the group's tail-needing records (ballot
// prefix); the last CTA to finish scans the per-group tail counts into group
// bases and reserves the tail blocks from the free list. A fork's tail block
// is free_list[cursor + tbase[g] + rank] — the (group, record)-order rank, as
// in the serial restatement.
__global__ void __launch_bounds__(kPlanWarps * 32)
fork_plan_kernel(const int32_t* forks, int group_cap, const int32_t* counts, int counts_stride,
                 int n_groups, int block_tokens, ForkWs ws, int32_t* free_cursor,
                 int free_list_len, int32_t* status) {
  __shared__ int sh[kScanThreads / 32];
  __shared__ int last;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * kPlanWarps + (threadIdx.x >> 5);
  if (g < n_groups) {
    const int c = group_count(counts, counts_stride, g, group_cap);
    int running = 0;
    for (int k0 = 0; k0 < c; k0 += 32) {
      const int k = k0 + lane;
      const int64_t rec = int64_t(g) * group_cap + k;
      const bool flag = k < c && (forks[rec * 4 + 3] % block_tokens) != 0;
      const unsigned m = __ballot_sync(0xffffffffu, flag);
      if (k < c) ws.rank[rec] = flag ? running + __popc(m & ((1u << lane) - 1u)) : -1;
      running += __popc(m);
    }
    if (lane == 0) {
      ws.gcount[g] = c;
      ws.gtail[g] = running;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ws.meta + 2, 1) == int(gridDim.x) - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // exclusive scan of the group tail counts (fixed group order)
  int base = 0;
  for (int g0 = 0; g0 < n_groups; g0 += blockDim.x) {
    const int gg = g0 + int(threadIdx.x);
    const int v = gg < n_groups ? __ldcg(ws.gtail + gg) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int warp = threadIdx.x >> 5;
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    int wbase = 0, total = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) {
      if (w < warp) wbase += sh[w];
      total += sh[w];
    }
    if (gg < n_groups) ws.tbase[gg] = base + wbase + x - v;
    base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int cursor = *free_cursor;
    ws.meta[0] = cursor;
    if (cursor + base > free_list_len) {
      if (status) status[0] = 1;
      ws.meta[1] = free_list_len - cursor;     // tails beyond the list are skipped
      *free_cursor = free_list_len;
    } else {
      if (status) status[0] = 0;
      ws.meta[1] = base;
      *free_cursor = cursor + base;
    }
    ws.meta[2] = 0;                            // ready for the next call
  }
}

// One CTA per (group, record) slot: copy the root's full blocks into the
// child's row (refcount += 1 each, order-independent), the reserved tail
// block + its KV bytes, -1 for the rest.
template <int UNROLL, bool STCS>
__global__ void __launch_bounds__(128)
fork_exec_kernel(const int32_t* forks, int rows_per_group, int group_cap, ForkWs ws,
                 int32_t* table, int table_stride, int32_t* refcount, const int32_t* free_list,
                 char* kv, int64_t kv_bytes_per_token, int block_tokens) {
  const int64_t rec = blockIdx.x;
  const int g = int(rec / group_cap), k = int(rec - int64_t(g) * group_cap);
  if (k >= ws.gcount[g]) return;
  const int32_t* fr = forks + rec * 4;
  const int child = fr[0], root = fr[2], prefix = fr[3];
  const int64_t gbase = int64_t(g) * rows_per_group;
  const int32_t* src = table + (gbase + root) * table_stride;
  int32_t* dst = table + (gbase + child) * table_stride;
  const int n_full = prefix / block_tokens;
  const int tail_tok = prefix - n_full * block_tokens;
  const int rank = ws.rank[rec];
  const int trank = rank >= 0 ? ws.tbase[g] + rank : -1;
  const bool has_tail = tail_tok > 0 && trank >= 0 && trank < ws.meta[1];
  const int tail_blk = has_tail ? free_list[ws.meta[0] + trank] : -1;
  for (int j = threadIdx.x; j < table_stride; j += blockDim.x) {
    int v = -1;
    if (j < n_full) {
      v = src[j];
      atomicAdd(&refcount[v], 1);
    } else if (j == n_full && tail_tok > 0) {
      v = tail_blk;
    }
    dst[j] = v;
  }
  if (!has_tail || kv == nullptr) {
    if (has_tail && threadIdx.x == 0) refcount[tail_blk] = 1;
    return;
  }
  if (threadIdx.x == 0) refcount[tail_blk] = 1;
  const int64_t block_bytes = kv_bytes_per_token * block_tokens;
  const char* s = kv + int64_t(src[n_full]) * block_bytes;
  char* d = kv + int64_t(tail_blk) * block_bytes;
  const int64_t nbytes = int64_t(tail_tok) * kv_bytes_per_token;
  if ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | uintptr_t(nbytes)) % 16 == 0) {
    const int64_t nv = nbytes / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    // UNROLL 16-byte loads per thread in flight before their stores
    for (int64_t i0 = 0; i0 < nv; i0 += UNROLL * 128) {
      uint4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t i = i0 + u * 128 + threadIdx.x;
        if (i < nv) v[u] = ldg_stream(s4 + i);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t i = i0 + u * 128 + threadIdx.x;
        if (i < nv) {
          if constexpr (STCS) __stcs(d4 + i, v[u]);
          else d4[i] = v[u];
        }
      }
    }
  } else {
    for (int64_t i = threadIdx.x; i < nbytes; i += blockDim.x) d[i] = s[i];
  }
}

// ---------------------------------------------------------------------------
// Segmented sort of unique 64-bit keys (level << 61 | arrival << 21 | order),
// one CTA per segment, bitonic in shared memory. Equals repeated
// next_request pops over one queue snapshot (scheduler.py:76-93) because the
// (level, arrival, order) keys are unique.
constexpr int kSortMax = 4096;

__global__ void __launch_bounds__(1024)
segsort_kernel(const uint64_t* keys, const int32_t* seg_off, int32_t* out_perm) {
  __shared__ uint64_t k[kSortMax];
  __shared__ int32_t v[kSortMax];
  const int seg = blockIdx.x;
  const int lo = seg_off[seg], n = seg_off[seg + 1] - lo;
  if (n > kSortMax) {   // segment too large for one CTA: flag every entry
    for (int i = threadIdx.x; i < n; i += blockDim.x) out_perm[lo + i] = -1;
    return;
  }
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    k[i] = i < n ? keys[lo + i] : ~0ull;
    v[i] = i < n ? i : 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = k[i] > k[j] || (k[i] == k[j] && v[i] > v[j]);
          if (gt == up) {
            const uint64_t tk = k[i]; k[i] = k[j]; k[j] = tk;
            const int32_t tv = v[i]; v[i] = v[j]; v[j] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out_perm[lo + i] = lo + v[i];
}

// ---------------------------------------------------------------------------
// Whole-queue sort for snapshots longer than one CTA's 4096 keys: (1) tiles of
// kSortMax keys bitonic-sorted in shared memory (segsort_kernel over uniform
// tiles, pairs (key, index) written to a ping-pong buffer); (2) merge passes
// doubling the run width, each output element placed by a merge-path search:
// thread t produces kMergeItems consecutive outputs of its pair of runs, finding
// where its diagonal crosses the two runs by binary search, then merging
// sequentially. Ordering is (key, index), so equal keys keep input order.
constexpr int kMergeThreads = 256, kMergeItems = 8;

__device__ __forceinline__ bool pair_less(uint64_t ka, int32_t ia, uint64_t kb, int32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(1024)
tile_sort_kernel(const uint64_t* keys, int64_t n, uint64_t* out_k, int32_t* out_i) {
  __shared__ uint64_t k[kSortMax];
  __shared__ int32_t v[kSortMax];
  const int64_t lo = int64_t(blockIdx.x) * kSortMax;
  const int cnt = int(n - lo < kSortMax ? n - lo : int64_t(kSortMax));
  int m = 1;
  while (m < cnt) m <<= 1;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    k[i] = i < cnt ? keys[lo + i] : ~0ull;
    v[i] = i < cnt ? int32_t(lo + i) : 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = pair_less(k[j], v[j], k[i], v[i]);
          if (gt == up) {
            const uint64_t tk = k[i]; k[i] = k[j]; k[j] = tk;
            const int32_t tv = v[i]; v[i] = v[j]; v[j] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    out_k[lo + i] = k[i];
    out_i[lo + i] = v[i];
  }
}

__global__ void __launch_bounds__(kMergeThreads)
merge_pass_kernel(const uint64_t* in_k, const int32_t* in_i, int64_t n, int64_t width,
                  uint64_t* out_k, int32_t* out_i) {
  const int64_t d0 = (int64_t(blockIdx.x) * kMergeThreads + threadIdx.x) * kMergeItems;
  if (d0 >= n) return;
  const int64_t pair = d0 / (2 * width);
  const int64_t a0 = pair * 2 * width;
  const int64_t a1 = a0 + width < n ? a0 + width : n, b1 = a0 + 2 * width < n ? a0 + 2 * width : n;
  const int64_t na = a1 - a0, nb = b1 - a1;
  const int64_t d = d0 - a0;                          // diagonal within the pair
  // merge path: the number i of A elements among the first d outputs
  int64_t lo = d - nb > 0 ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int64_t i = (lo + hi) >> 1;                 // A[i] vs B[d - 1 - i]
    const int64_t j = d - 1 - i;
    if (pair_less(in_k[a1 + j], in_i[a1 + j], in_k[a0 + i], in_i[a0 + i])) hi = i;
    else lo = i + 1;
  }
  int64_t i = lo, j = d - lo;
  const int64_t end = d0 + kMergeItems < b1 ? d0 + kMergeItems : b1;
  for (int64_t o = d0; o < end; ++o) {
    bool take_a;
    if (i >= na) take_a = false;
    else if (j >= nb) take_a = true;
    else take_a = !pair_less(in_k[a1 + j], in_i[a1 + j], in_k[a0 + i], in_i[a0 + i]);
    if (take_a) { out_k[o] = in_k[a0 + i]; out_i[o] = in_i[a0 + i]; ++i; }
    else        { out_k[o] = in_k[a1 + j]; out_i[o] = in_i[a1 + j]; ++j; }
  }
}

}  // namespace duchess

using namespace duchess;

extern "C" size_t duchess_sort_keys_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return size_t(n) * 2 * (sizeof(uint64_t) + sizeof(int32_t)) + 64;
}

extern "C" int duchess_sort_keys(const uint64_t* keys, int64_t n, int32_t* out_perm,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || (n > 0 && (!keys || !out_perm))) return DUCHESS_EINVAL;
  if (n > INT32_MAX) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  if (!workspace || workspace_bytes < duchess_sort_keys_workspace_bytes(n)) return DUCHESS_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t* k0 = static_cast<uint64_t*>(workspace);
  uint64_t* k1 = k0 + n;
  int32_t* i0 = reinterpret_cast<int32_t*>(k1 + n);
  int32_t* i1 = i0 + n;
  tile_sort_kernel<<<unsigned((n + kSortMax - 1) / kSortMax), 1024, 0, s>>>(keys, n, k0, i0);
  const unsigned grid = unsigned((n + int64_t(kMergeThreads) * kMergeItems - 1) /
                                 (int64_t(kMergeThreads) * kMergeItems));
  for (int64_t w = kSortMax; w < n; w <<= 1) {
    merge_pass_kernel<<<grid, kMergeThreads, 0, s>>>(k0, i0, n, w, k1, i1);
    std::swap(k0, k1);
    std::swap(i0, i1);
  }
  cudaMemcpyAsync(out_perm, i0, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" size_t duchess_fork_workspace_bytes(int32_t n_groups, int32_t group_cap) {
  if (n_groups < 0 || group_cap < 0) return 0;
  const size_t nf = size_t(n_groups) * size_t(group_cap);
  return (3 * size_t(n_groups) + nf + 4) * sizeof(int32_t);
}

extern "C" int duchess_fork_cow(const int32_t* forks, int32_t group_cap, const int32_t* group_counts,
                                int32_t counts_stride, int32_t n_groups, int32_t rows_per_group,
                                int32_t* block_table, int32_t table_stride, int32_t* refcount,
                                const int32_t* free_list, int32_t free_list_len,
                                int32_t* free_cursor, void* kv_pool, int64_t kv_bytes_per_token,
                                int32_t block_tokens, int32_t* status, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (n_groups < 0 || group_cap < 0 || block_tokens < 1 || table_stride < 1) return DUCHESS_EINVAL;
  if (!forks || !block_table || !refcount || !free_cursor) return DUCHESS_EINVAL;
  if (kv_pool && kv_bytes_per_token < 1) return DUCHESS_EINVAL;
  if (n_groups == 0 || group_cap == 0) return DUCHESS_OK;
  if (!workspace || workspace_bytes < duchess_fork_workspace_bytes(n_groups, group_cap))
    return DUCHESS_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nf = size_t(n_groups) * size_t(group_cap);
  int32_t* w = static_cast<int32_t*>(workspace);
  ForkWs ws{w, w + n_groups, w + 2 * int64_t(n_groups), w + 3 * int64_t(n_groups),
            w + 3 * int64_t(n_groups) + int64_t(nf)};
  fork_plan_kernel<<<unsigned((n_groups + kPlanWarps - 1) / kPlanWarps), kPlanWarps * 32, 0, s>>>(
      forks, group_cap, group_counts, counts_stride, n_groups, block_tokens, ws, free_cursor,
      free_list_len, status);
  // tail-copy loads in flight per thread (env DUCHESS_K3_UNROLL, for sweeps;
  // C4 with write-back stores: 4 -> 0.857, 8 -> 0.849, 16 -> 0.66 of the copy peak)
  static const int unroll = [] { const char* e = getenv("DUCHESS_K3_UNROLL"); return e ? atoi(e) : 4; }();
  // tail-copy stores: write-back (default; C4 142 vs 138 M forks/s with streaming
  // .cs stores, env DUCHESS_K3_WB=0)
  static const bool wb = [] { const char* e = getenv("DUCHESS_K3_WB"); return e ? atoi(e) != 0 : true; }();
  auto k = wb ? (unroll >= 16 ? fork_exec_kernel<16, false> : unroll >= 8 ? fork_exec_kernel<8, false>
                                                            : fork_exec_kernel<4, false>)
              : (unroll >= 16 ? fork_exec_kernel<16, true> : unroll >= 8 ? fork_exec_kernel<8, true>
                                                           : fork_exec_kernel<4, true>);
  k<<<unsigned(nf), 128, 0, s>>>(forks, rows_per_group, group_cap, ws, block_table, table_stride,
                                 refcount, free_list, static_cast<char*>(kv_pool),
                                 kv_bytes_per_token, block_tokens);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_sort_difficulty(const uint64_t* keys, const int32_t* seg_offsets,
                                       int32_t n_segs, int32_t* out_perm, void* stream) {
  if (n_segs < 0 || !keys || !seg_offsets || !out_perm) return DUCHESS_EINVAL;
  if (n_segs == 0) return DUCHESS_OK;
  segsort_kernel<<<unsigned(n_segs), 1024, 0, static_cast<cudaStream_t>(stream)>>>(keys, seg_offsets,
                                                                                   out_perm);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
