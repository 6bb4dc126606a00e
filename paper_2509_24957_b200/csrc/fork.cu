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
#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kPlanThreads = 1024;

__device__ __forceinline__ int group_count(const int32_t* counts, int stride, int g, int cap) {
  return counts ? min(max(counts[int64_t(g) * stride], 0), cap) : cap;
}

// Block-wide exclusive scan (1024 threads) of one int per thread.
__device__ __forceinline__ int block_excl_scan(int v, int* total, int* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < (kPlanThreads / 32) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;   // inclusive warp totals
  }
  __syncthreads();
  const int warp_base = warp ? sh[warp - 1] : 0;
  *total = sh[kPlanThreads / 32 - 1];
  __syncthreads();
  return warp_base + x - v;
}

// Plan: group bases (scan of counts), per-fork (group, record) map and tail rank.
__global__ void __launch_bounds__(kPlanThreads)
fork_plan_kernel(const int32_t* forks, int group_cap, const int32_t* counts, int counts_stride,
                 int n_groups, int block_tokens, int32_t* ws_base, int32_t* ws_map,
                 int32_t* ws_tail, int32_t* ws_meta, int32_t* free_cursor, int free_list_len,
                 int32_t* status) {
  __shared__ int sh[32];
  int running = 0;
  for (int g0 = 0; g0 < n_groups; g0 += kPlanThreads) {
    const int g = g0 + threadIdx.x;
    const int c = g < n_groups ? group_count(counts, counts_stride, g, group_cap) : 0;
    int total;
    const int ex = block_excl_scan(c, &total, sh);
    if (g < n_groups) ws_base[g] = running + ex;
    running += total;
  }
  const int n_forks = running;
  if (threadIdx.x == 0) ws_base[n_groups] = n_forks;
  __syncthreads();
  int tails = 0;
  for (int f0 = 0; f0 < n_forks; f0 += kPlanThreads) {
    const int f = f0 + threadIdx.x;
    int flag = 0, rec = -1;
    if (f < n_forks) {
      int lo = 0, hi = n_groups;                 // last g with base[g] <= f
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ws_base[mid] <= f) lo = mid; else hi = mid;
      }
      rec = lo * group_cap + (f - ws_base[lo]);
      flag = (forks[int64_t(rec) * 4 + 3] % block_tokens) != 0;
      ws_map[f] = rec;
    }
    int total;
    const int ex = block_excl_scan(flag, &total, sh);
    if (f < n_forks) ws_tail[f] = flag ? tails + ex : -1;
    tails += total;
  }
  if (threadIdx.x == 0) {
    const int cursor = *free_cursor;
    ws_meta[0] = n_forks;
    ws_meta[1] = cursor;
    if (cursor + tails > free_list_len) {
      if (status) status[0] = 1;
      ws_meta[2] = free_list_len - cursor;     // tails beyond the list are skipped
      *free_cursor = free_list_len;
    } else {
      if (status) status[0] = 0;
      ws_meta[2] = tails;
      *free_cursor = cursor + tails;
    }
  }
}

__global__ void __launch_bounds__(128)
fork_exec_kernel(const int32_t* forks, int rows_per_group, int group_cap, const int32_t* ws_map,
                 const int32_t* ws_tail, const int32_t* ws_meta, int32_t* table, int table_stride,
                 int32_t* refcount, const int32_t* free_list, char* kv,
                 int64_t kv_bytes_per_token, int block_tokens) {
  const int f = blockIdx.x;
  if (f >= ws_meta[0]) return;
  const int rec = ws_map[f];
  const int g = rec / group_cap;
  const int32_t* fr = forks + int64_t(rec) * 4;
  const int child = fr[0], root = fr[2], prefix = fr[3];
  const int64_t gbase = int64_t(g) * rows_per_group;
  const int32_t* src = table + (gbase + root) * table_stride;
  int32_t* dst = table + (gbase + child) * table_stride;
  const int n_full = prefix / block_tokens;
  const int tail_tok = prefix - n_full * block_tokens;
  const int rank = ws_tail[f];
  const bool has_tail = tail_tok > 0 && rank >= 0 && rank < ws_meta[2];
  const int tail_blk = has_tail ? free_list[ws_meta[1] + rank] : -1;
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
    int64_t i = threadIdx.x;
    for (; i + 3 * 128 < nv; i += 4 * 128) {
      const uint4 a = ldg_stream(s4 + i), b = ldg_stream(s4 + i + 128);
      const uint4 c = ldg_stream(s4 + i + 256), e = ldg_stream(s4 + i + 384);
      __stcs(d4 + i, a); __stcs(d4 + i + 128, b); __stcs(d4 + i + 256, c); __stcs(d4 + i + 384, e);
    }
    for (; i < nv; i += 128) __stcs(d4 + i, ldg_stream(s4 + i));
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

}  // namespace duchess

using namespace duchess;

extern "C" size_t duchess_fork_workspace_bytes(int32_t n_groups, int32_t group_cap) {
  if (n_groups < 0 || group_cap < 0) return 0;
  const size_t nf = size_t(n_groups) * size_t(group_cap);
  return (size_t(n_groups) + 1 + 2 * nf + 4) * sizeof(int32_t);
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
  int32_t* ws_base = static_cast<int32_t*>(workspace);
  int32_t* ws_map = ws_base + n_groups + 1;
  int32_t* ws_tail = ws_map + nf;
  int32_t* ws_meta = ws_tail + nf;
  fork_plan_kernel<<<1, kPlanThreads, 0, s>>>(forks, group_cap, group_counts, counts_stride,
                                             n_groups, block_tokens, ws_base, ws_map, ws_tail,
                                             ws_meta, free_cursor, free_list_len, status);
  fork_exec_kernel<<<unsigned(nf), 128, 0, s>>>(forks, rows_per_group, group_cap, ws_map, ws_tail,
                                                ws_meta, block_table, table_stride, refcount,
                                                free_list, static_cast<char*>(kv_pool),
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
