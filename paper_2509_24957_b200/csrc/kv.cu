// K3 in the round: a persistent paged KV cache driven by the engine's rounds.
//
// The reference forks by pure accounting — the child resumes the next
// template at the parent's position without re-charging the prefix
// (orchestrator.py:254-268 _spawn(offset_base=source.position), :378-388) —
// and the paper serves that with vLLM prefix caching. Here the
// prefix lives in a paged KV cache and a fork is a copy-on-write block-table
// duplication, applied every round right after duchess_round:
//
//   1. forks of the round just decided (DuchessState.forks, record order): the
//      child's row takes the root's first prefix/bt blocks (refcount += 1) and
//      a private block holding a copy of the partial tail (prefix % bt tokens
//      of KV bytes, copied by the slot's warp; also listed in `jobs`);
//   2. releases: every row still holding blocks whose branch is no longer
//      active (early-terminated, natural end, capped, cancelled) drops its
//      references; a block whose refcount reaches 0 goes back to the free stack;
//   3. appends: every active branch's row grows to ceil(position / bt) blocks
//      (the tokens decoded this round; the LLM writes their KV, this kernel
//      only provides the blocks).
//   A request that finished this round (round record `done`) has its whole
//   arena reset; its successor in the slot starts from an empty arena.
//
// Allocation is per request slot: slot r owns blocks [r*P, (r+1)*P) of the
// pool (an arena, P = blocks_per_slot) with a LIFO free stack plus a
// high-water mark, so one warp per slot does all of its bookkeeping with no
// atomics, and a request's block tables are a pure function of its own
// rounds (the CPU restatement, oracle/kvcache.py, replays the oracle
// DuchessRun's actions and matches tables, refcounts and stacks exactly).
// Within a slot the order is fixed: forks in record order, releases by
// branch id then block index, appends by branch id then block index.
#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kKvWarps = 4;
constexpr int kArTop = 0, kArHwm = 1, kArOwner = 2, kArPeak = 3;
constexpr int kWin = 16;         // entries per lane per window (512 per warp)

// Shared-memory words per warp: per-branch tokens covered / status /
// position / entry offsets. Kept small (1 KB at 64 branch ids) so the kernel's
// CTAs fit beside a persistent scorer's on every SM: K1 assigns its units to
// CTAs statically, so a CTA kept waiting for shared memory would delay the
// whole scoring launch of the other request shard.
__host__ __device__ inline int64_t kv_warp_words(int B) { return 4 * int64_t(B) + 4; }

// Warp-wide byte copy (global -> global): 16-byte streaming loads / stores,
// eight in flight per lane when both ends and the size are 16-byte aligned.
__device__ __forceinline__ void kv_copy_bytes(const char* sp, char* dp, int64_t nbytes, int lane) {
  if (((reinterpret_cast<uintptr_t>(sp) | reinterpret_cast<uintptr_t>(dp) | uintptr_t(nbytes)) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(sp);
    uint4* d4 = reinterpret_cast<uint4*>(dp);
    const int64_t nv = nbytes / 16;
    for (int64_t i0 = 0; i0 < nv; i0 += 8 * 32) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = i0 + u * 32 + lane;
        if (i < nv) v[u] = ldg_stream(s4 + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = i0 + u * 32 + lane;
        if (i < nv) __stcs(d4 + i, v[u]);
      }
    }
  } else {
    for (int64_t i = lane; i < nbytes; i += 32) dp[i] = sp[i];
  }
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// One warp per request slot; the slot's arena (refcounts, free stack, block
// table rows) lives in global memory (L2-resident: a few KB per slot) and
// only this warp touches it, so every phase is a wave of independent loads
// and stores over 32-entry chunks rather than a chain of dependent accesses:
// the branch fields and fork records are read in one wave, the released rows'
// entries in one window of 512, the blocks the appends pop in one wave.
__global__ void __launch_bounds__(kKvWarps * 32)
kv_round_kernel(DuchessPolicy pol, DuchessState s, DuchessKV kv) {
  extern __shared__ int32_t kv_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int r = blockIdx.x * (blockDim.x >> 5) + wib;
  // Overlapped launch (DUCHESS_KV_OVERLAP): this grid runs beside the
  // preceding kernel (the next round's scorer, which does not touch what is
  // read here) and waits for it only at the end, so the next duchess_round,
  // chained behind this grid, still sees the scorer's results.
  pdl_launch_dependents();
  if (r >= s.n_slots) {
    pdl_wait();
    return;
  }
  const int B = s.branch_cap, C = pol.max_branches, NB = kv.max_blocks, bt = kv.block_tokens;
  const int P = kv.blocks_per_slot;
  int32_t* bk = kv_smem + int64_t(wib) * kv_warp_words(B);        // [B] tokens covered
  int32_t* bs = bk + B;                                            // [B] status
  int32_t* bp = bs + B;                                            // [B] position
  int32_t* bo = bp + B;                                            // [B + 1] entry offsets
  const int base = r * P;
  const int64_t rB = int64_t(r) * B;
  int32_t* ref = kv.refcount + int64_t(r) * P;                     // by local block id
  int32_t* stk = kv.free_stack + int64_t(r) * P;
  int32_t* g_ar = kv.arena + int64_t(r) * 4;
  int32_t* jobs = kv.jobs + int64_t(r) * C * 4;
  auto row = [&](int b) { return kv.table + (rB + b) * NB; };
  const int32_t* rec = s.round_rec + int64_t(r) * DUCHESS_REC_WORDS;
  const bool decided = rec[DUCHESS_REC_ROUND] != 0;
  const bool finished = decided && rec[DUCHESS_REC_DONE] != 0;
  const int nf = decided ? rec[DUCHESS_REC_NFORKS] : 0;
  int top = g_ar[kArTop], hwm = g_ar[kArHwm], owner = g_ar[kArOwner], peak = g_ar[kArPeak];
  const int req = s.done[r] ? -1 : s.slot_req[r];
  const int nb = req >= 0 || decided ? s.n_branches[r] : 0;
  int overflow = 0, n_alloc = 0, n_free = 0, n_jobs = 0;   // warp-uniform
  int ovl = 0;                                              // per lane
  long long tail_bytes = 0;
  const bool reset = finished || (owner >= 0 && owner != req);

  // branch fields (two branches per lane per round trip)
  for (int b0 = 0; b0 < nb; b0 += 64) {
    const int b1 = b0 + lane, b2 = b0 + 32 + lane;
    int st1 = 0, st2 = 0, o1 = 0, o2 = 0, d1 = 0, d2 = 0, k1 = 0, k2 = 0;
    if (b1 < nb) { st1 = s.br_status[rB + b1]; o1 = s.br_offset[rB + b1]; d1 = s.br_decoded[rB + b1]; k1 = kv.kv_tokens[rB + b1]; }
    if (b2 < nb) { st2 = s.br_status[rB + b2]; o2 = s.br_offset[rB + b2]; d2 = s.br_decoded[rB + b2]; k2 = kv.kv_tokens[rB + b2]; }
    if (b1 < nb) { bs[b1] = st1; bp[b1] = o1 + d1; bk[b1] = reset ? 0 : k1; }
    if (b2 < nb) { bs[b2] = st2; bp[b2] = o2 + d2; bk[b2] = reset ? 0 : k2; }
  }

  if (reset) {
    // the arena's request is gone: clear every row it held, zero its refcounts
    for (int b0 = 0; b0 < B; b0 += 32) {
      const int b = b0 + lane;
      const int have = b < B ? (kv.kv_tokens[rB + b] + bt - 1) / bt : 0;
      if (have > 0) kv.kv_tokens[rB + b] = 0;
      unsigned m = __ballot_sync(0xffffffffu, have > 0);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int hb = __shfl_sync(0xffffffffu, have, src);
        int32_t* t = row(b0 + src);
        for (int j = lane; j < hb; j += 32) t[j] = -1;
      }
    }
    for (int j = lane; j < hwm; j += 32) ref[j] = 0;
    n_free = hwm;
    top = 0;
    hwm = 0;
    owner = -1;
  }
  __syncwarp();

  if (!reset && decided) {
    // 1. forks of the round just decided, in record order
    int fc = -1, fr_ = -1, fp = 0;                    // lane f holds fork f's record
    if (lane < nf) {
      const int32_t* fr = s.forks + (int64_t(r) * C + lane) * 4;
      fc = fr[0];
      fr_ = fr[2];
      fp = fr[3];
    }
    for (int f = 0; f < nf; ++f) {
      int child, root, prefix;
      if (f < 32) {
        child = __shfl_sync(0xffffffffu, fc, f);
        root = __shfl_sync(0xffffffffu, fr_, f);
        prefix = __shfl_sync(0xffffffffu, fp, f);
      } else {
        const int32_t* fr = s.forks + (int64_t(r) * C + f) * 4;
        child = fr[0];
        root = fr[2];
        prefix = fr[3];
      }
      if (bs[child] != DUCHESS_ACTIVE) continue;              // cancelled / ended at once
      const int n_full = prefix / bt, tail = prefix - n_full * bt;
      const int32_t* src = row(root);
      int32_t* dst = row(child);
      for (int j = lane; j < n_full; j += 32) {
        const int blk = src[j];
        dst[j] = blk;
        if (blk >= 0) atomicAdd(ref + (blk - base), 1);        // distinct within a row
      }
      if (tail > 0) {
        int blk = -1;
        if (top > 0) blk = stk[--top];
        else if (hwm < P) blk = hwm++;
        else ++overflow;
        if (blk >= 0) {
          ++n_alloc;
          ++n_jobs;
          tail_bytes += (long long)(tail) * kv.kv_bytes_per_token;
        }
        if (lane == 0) {
          dst[n_full] = blk < 0 ? -1 : blk + base;
          if (blk >= 0) {
            ref[blk] = 1;
            int32_t* jb = jobs + (n_jobs - 1) * 4;
            jb[0] = src[n_full];                              // the root's block with the tail
            jb[1] = blk + base;
            jb[2] = tail;
          }
        }
        if (blk >= 0 && kv.kv_pool) {
          // copy the partial tail's KV bytes (warp-wide 16-byte streams,
          // 8 in flight per lane); tails average a few KB
          const int sblk = __shfl_sync(0xffffffffu, lane == 0 ? src[n_full] : 0, 0);
          const int64_t block_bytes = kv.kv_bytes_per_token * bt;
          kv_copy_bytes(kv.kv_pool + int64_t(sblk) * block_bytes,
                        kv.kv_pool + int64_t(blk + base) * block_bytes,
                        int64_t(tail) * kv.kv_bytes_per_token, lane);
        }
      }
      if (lane == 0) bk[child] = prefix;
      __syncwarp();
    }
    // 2. releases in (branch id, block index) order. The released rows'
    // entries are flattened in that order, read (and cleared to -1 in the
    // table) a window of 512 at a time — lane l holds entries l, l+32, ... —
    // then walked 32 at a time. Rows may share blocks, so equal blocks within
    // a chunk are merged on their last lane, which alone sees the count reach
    // zero (as walking the entries one by one would).
    int total = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const int h = (b < nb && bs[b] != DUCHESS_ACTIVE) ? (bk[b] + bt - 1) / bt : 0;
      int tot;
      const int off = warp_excl_scan(h, lane, tot);
      if (b < nb) bo[b] = total + off;
      total += tot;
    }
    __syncwarp();
    auto entry_row = [&](int e) {                     // last b with bo[b] <= e
      int lo = 0, hi = nb - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (bo[mid] <= e) lo = mid; else hi = mid - 1;
      }
      return lo;
    };
    for (int w0 = 0; w0 < total; w0 += kWin * 32) {
      int v[kWin];
#pragma unroll
      for (int u = 0; u < kWin; ++u) {
        const int e = w0 + u * 32 + lane;
        v[u] = -1;
        if (e < total) {
          const int b = entry_row(e);
          int32_t* t = row(b) + (e - bo[b]);
          v[u] = *t;
          *t = -1;
        }
      }
#pragma unroll
      for (int u = 0; u < kWin; ++u) {
        if (w0 + u * 32 >= total) break;
        const int loc = v[u] < 0 ? -1 : v[u] - base;
        const unsigned grp = __match_any_sync(0xffffffffu, loc);
        bool freed = false;
        if (loc >= 0 && (grp >> lane) == 1u) freed = atomicSub(ref + loc, __popc(grp)) == __popc(grp);
        const unsigned m = __ballot_sync(0xffffffffu, freed);
        if (freed) stk[top + __popc(m & ((1u << lane) - 1u))] = loc;
        top += __popc(m);
        n_free += __popc(m);
      }
    }
    for (int b = lane; b < nb; b += 32)
      if (bs[b] != DUCHESS_ACTIVE) bk[b] = 0;
    __syncwarp();
  }

  // 3. appends: every active row grows to ceil(position / bt) blocks; the
  // allocation sequence is (branch id, block index), one lane per block
  if (req >= 0) {
    owner = req;
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      int add = 0;
      if (b < nb && bs[b] == DUCHESS_ACTIVE) {
        const int want = (bp[b] + bt - 1) / bt;
        const int need = min(want, NB);
        ovl += want - need;                          // position beyond the table width
        add = max(0, need - (bk[b] + bt - 1) / bt);
      }
      int tot;
      const int off = warp_excl_scan(add, lane, tot);
      if (b < nb) bo[b] = run + off;
      run += tot;
    }
    __syncwarp();
    const int m = run;
    for (int a = lane; a < m; a += 32) {
      int lo = 0, hi = nb - 1;                               // last b with bo[b] <= a
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (bo[mid] <= a) lo = mid; else hi = mid - 1;
      }
      const int b = lo;
      const int j = (bk[b] + bt - 1) / bt + (a - bo[b]);
      int blk = -1;
      if (a < top) blk = stk[top - 1 - a];
      else if (hwm + (a - top) < P) blk = hwm + (a - top);
      row(b)[j] = blk < 0 ? -1 : blk + base;
      if (blk >= 0) ref[blk] = 1;
    }
    const int from_stack = min(m, top);
    const int fresh = min(m - from_stack, P - hwm);
    overflow += m - from_stack - fresh;
    n_alloc += from_stack + fresh;
    top -= from_stack;
    hwm += fresh;
    __syncwarp();
    for (int b = lane; b < nb; b += 32)
      if (bs[b] == DUCHESS_ACTIVE) bk[b] = bp[b];
    __syncwarp();
  }

  for (int b = lane; b < nb; b += 32) kv.kv_tokens[rB + b] = bk[b];
  peak = max(peak, hwm);
  overflow += __reduce_add_sync(0xffffffffu, ovl);
  if (lane == 0) {
    g_ar[kArTop] = top;
    g_ar[kArHwm] = hwm;
    g_ar[kArOwner] = owner;
    g_ar[kArPeak] = peak;
    kv.job_count[r] = n_jobs;
    if (n_alloc) add_counter(&kv.counters[DUCHESS_KV_CNT_ALLOC], n_alloc);
    if (n_free) add_counter(&kv.counters[DUCHESS_KV_CNT_FREE], n_free);
    if (n_jobs) add_counter(&kv.counters[DUCHESS_KV_CNT_TAIL_BYTES], tail_bytes);
    if (overflow) add_counter(&kv.counters[DUCHESS_KV_CNT_OVERFLOW], overflow);
  }
  pdl_wait();
}

}  // namespace duchess

using namespace duchess;

extern "C" int duchess_kv_round(const DuchessPolicy* policy, const DuchessState* state,
                                const DuchessKV* kv, void* stream) {
  if (!policy || !state || !kv) return DUCHESS_EINVAL;
  if (kv->block_tokens < 1 || kv->blocks_per_slot < 1 || kv->max_blocks < 1) return DUCHESS_EINVAL;
  if (!kv->table || !kv->kv_tokens || !kv->refcount || !kv->free_stack || !kv->arena ||
      !kv->jobs || !kv->job_count || !kv->counters)
    return DUCHESS_EINVAL;
  if (kv->kv_pool && kv->kv_bytes_per_token < 1) return DUCHESS_EINVAL;
  if (int64_t(state->n_slots) * kv->blocks_per_slot > INT32_MAX) return DUCHESS_EINVAL;
  if (!state->round_rec || !state->forks || !state->br_status || !state->n_branches)
    return DUCHESS_EINVAL;
  if (state->n_slots == 0) return DUCHESS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t per_warp = size_t(kv_warp_words(state->branch_cap)) * 4;
  const int warps = int(per_warp * kKvWarps <= 200 * 1024 ? kKvWarps : 200 * 1024 / per_warp);
  if (warps < 1) return DUCHESS_EINVAL;                       // arena too large to stage
  const size_t smem = per_warp * warps;
  cudaFuncSetAttribute(kv_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned((state->n_slots + warps - 1) / warps));
  cfg.blockDim = dim3(warps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (kv->flags & DUCHESS_KV_OVERLAP) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kv_round_kernel, *policy, *state, *kv);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
