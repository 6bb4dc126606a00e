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
//      of KV bytes; a "tail job" for the copy kernel);
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

struct KvSlot {
  const DuchessKV& kv;
  int32_t* stack;     // this slot's free stack [P]
  int32_t* ref;       // this slot's refcounts [P] (local block ids)
  int32_t* ar;        // this slot's arena words
  int32_t base;       // r * P (global id of local block 0)
};

// Pop n blocks (lane j < n takes the j-th, as a global id): stack top first,
// then fresh blocks above the high-water mark; -1 (and an overflow count) past P.
__device__ __forceinline__ int kv_alloc(const KvSlot& k, int n, int j, int lane, int& top, int& hwm,
                                        int& overflow) {
  int blk = -1;
  if (j < n) {
    if (j < top) {
      blk = k.stack[top - 1 - j];
    } else {
      const int f = hwm + (j - top);
      if (f < k.kv.blocks_per_slot) blk = f;
    }
  }
  const int from_stack = min(n, top);
  const int fresh = min(n - from_stack, k.kv.blocks_per_slot - hwm);
  overflow += n - from_stack - fresh;
  top -= from_stack;
  hwm += fresh;
  (void)lane;
  return blk < 0 ? -1 : blk + k.base;          // global block id
}

__global__ void __launch_bounds__(kKvWarps * 32)
kv_round_kernel(DuchessPolicy pol, DuchessState s, DuchessKV kv) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kKvWarps + (threadIdx.x >> 5);
  if (r >= s.n_slots) return;
  const int B = s.branch_cap, C = pol.max_branches, NB = kv.max_blocks, bt = kv.block_tokens;
  const int P = kv.blocks_per_slot;
  KvSlot k{kv, kv.free_stack + int64_t(r) * P, kv.refcount + int64_t(r) * P,
           kv.arena + int64_t(r) * 4, r * P};
  const int64_t rB = int64_t(r) * B;
  int32_t* jobs = kv.jobs + int64_t(r) * C * 4;
  const int32_t* rec = s.round_rec + int64_t(r) * DUCHESS_REC_WORDS;
  const bool decided = rec[DUCHESS_REC_ROUND] != 0;
  const bool finished = decided && rec[DUCHESS_REC_DONE] != 0;
  int top = k.ar[kArTop], hwm = k.ar[kArHwm], owner = k.ar[kArOwner], peak = k.ar[kArPeak];
  const int req = s.done[r] ? -1 : s.slot_req[r];
  int overflow = 0, n_alloc = 0, n_free = 0, n_jobs = 0;
  long long tail_bytes = 0;
  auto row = [&](int b) { return kv.table + (rB + b) * NB; };

  if (finished || (owner >= 0 && owner != req)) {
    // the arena's request is gone: clear its rows, refcounts and stack
    for (int b = 0; b < B; ++b) {
      const int have = (kv.kv_tokens[rB + b] + bt - 1) / bt;
      if (have == 0) continue;
      int32_t* t = row(b);
      for (int j = lane; j < have; j += 32) t[j] = -1;
      if (lane == 0) kv.kv_tokens[rB + b] = 0;
    }
    for (int j = lane; j < hwm; j += 32) k.ref[j] = 0;
    n_free = hwm;
    top = 0;
    hwm = 0;
    owner = -1;
    __syncwarp();
  } else if (decided) {
    // 1. forks of the round just decided, in record order
    const int nf = rec[DUCHESS_REC_NFORKS];
    for (int f = 0; f < nf; ++f) {
      const int32_t* fr = s.forks + (int64_t(r) * C + f) * 4;
      const int child = fr[0], root = fr[2], prefix = fr[3];
      if (s.br_status[rB + child] != DUCHESS_ACTIVE) continue;   // cancelled / ended at once
      const int n_full = prefix / bt, tail = prefix - n_full * bt;
      const int32_t* src = row(root);
      int32_t* dst = row(child);
      for (int j = lane; j < n_full; j += 32) {
        const int blk = src[j];
        dst[j] = blk;
        if (blk >= 0) k.ref[blk - k.base] += 1;
      }
      if (tail > 0) {
        const int blk = __shfl_sync(0xffffffffu, kv_alloc(k, 1, lane, lane, top, hwm, overflow), 0);
        n_alloc += blk >= 0;
        if (lane == 0) {
          dst[n_full] = blk;
          if (blk >= 0) {
            k.ref[blk - k.base] = 1;
            int32_t* jb = jobs + n_jobs * 4;
            jb[0] = src[n_full];       // the root's block holding the partial tail
            jb[1] = blk;
            jb[2] = tail;
          }
        }
        if (blk >= 0) {
          ++n_jobs;
          tail_bytes += (long long)(tail) * kv.kv_bytes_per_token;
        }
      }
      if (lane == 0) kv.kv_tokens[rB + child] = prefix;
      __syncwarp();
    }
    // 2. releases: rows holding blocks whose branch is no longer active
    const int nb = s.n_branches[r];
    for (int b = 0; b < nb; ++b) {
      const int have = (kv.kv_tokens[rB + b] + bt - 1) / bt;
      if (have == 0 || s.br_status[rB + b] == DUCHESS_ACTIVE) continue;
      int32_t* t = row(b);
      for (int j0 = 0; j0 < have; j0 += 32) {
        const int j = j0 + lane;
        bool freed = false;
        int loc = -1;
        if (j < have) {
          const int blk = t[j];
          t[j] = -1;
          if (blk >= 0) {
            loc = blk - k.base;
            freed = --k.ref[loc] == 0;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, freed);
        if (freed) k.stack[top + __popc(m & ((1u << lane) - 1u))] = loc;
        top += __popc(m);
        n_free += __popc(m);
      }
      if (lane == 0) kv.kv_tokens[rB + b] = 0;
      __syncwarp();
    }
  }
  // 3. appends: active rows grow to the blocks their position needs
  if (req >= 0) {
    owner = req;
    const int nb = s.n_branches[r];
    for (int b = 0; b < nb; ++b) {
      if (s.br_status[rB + b] != DUCHESS_ACTIVE) continue;
      const int pos = s.br_offset[rB + b] + s.br_decoded[rB + b];
      const int have = (kv.kv_tokens[rB + b] + bt - 1) / bt;
      const int want = (pos + bt - 1) / bt;
      const int need = min(want, NB);
      overflow += want - need;                       // position beyond the table width
      if (need > have) {
        int32_t* t = row(b);
        for (int j0 = have; j0 < need; j0 += 32) {
          const int n = min(32, need - j0);
          const int blk = kv_alloc(k, n, lane, lane, top, hwm, overflow);
          if (lane < n) {
            t[j0 + lane] = blk;
            if (blk >= 0) k.ref[blk - k.base] = 1;
          }
          n_alloc += __popc(__ballot_sync(0xffffffffu, lane < n && blk >= 0));
        }
      }
      if (lane == 0) kv.kv_tokens[rB + b] = pos;
      __syncwarp();
    }
  }
  peak = max(peak, hwm);
  if (lane == 0) {
    k.ar[kArTop] = top;
    k.ar[kArHwm] = hwm;
    k.ar[kArOwner] = owner;
    k.ar[kArPeak] = peak;
    kv.job_count[r] = n_jobs;
    if (n_alloc) add_counter(&kv.counters[DUCHESS_KV_CNT_ALLOC], n_alloc);
    if (n_free) add_counter(&kv.counters[DUCHESS_KV_CNT_FREE], n_free);
    if (n_jobs) add_counter(&kv.counters[DUCHESS_KV_CNT_TAIL_BYTES], tail_bytes);
    if (overflow) add_counter(&kv.counters[DUCHESS_KV_CNT_OVERFLOW], overflow);
  }
}

// Tail copies of the round's forks: CTA-strided over the R*C job slots (slot
// r's first job_count[r] entries), 16-byte streaming loads and stores, four
// in flight per thread. Destinations are distinct fresh blocks, so job order
// does not matter.
__global__ void __launch_bounds__(256) kv_copy_kernel(DuchessKV kv, int n_slots, int C) {
  const int64_t block_bytes = kv.kv_bytes_per_token * kv.block_tokens;
  for (int64_t e = blockIdx.x; e < int64_t(n_slots) * C; e += gridDim.x) {
    const int r = int(e / C), q = int(e - int64_t(r) * C);
    if (q >= kv.job_count[r]) continue;
    const int32_t* jb = kv.jobs + e * 4;
    const char* sp = kv.kv_pool + int64_t(jb[0]) * block_bytes;
    char* dp = kv.kv_pool + int64_t(jb[1]) * block_bytes;
    const int64_t nbytes = int64_t(jb[2]) * kv.kv_bytes_per_token;
    if (((reinterpret_cast<uintptr_t>(sp) | reinterpret_cast<uintptr_t>(dp) | uintptr_t(nbytes)) & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(sp);
      uint4* d4 = reinterpret_cast<uint4*>(dp);
      const int64_t nv = nbytes / 16;
      int64_t i = threadIdx.x;
      for (; i + 3 * 256 < nv; i += 4 * 256) {
        const uint4 a = ldg_stream(s4 + i), b = ldg_stream(s4 + i + 256);
        const uint4 c = ldg_stream(s4 + i + 512), d = ldg_stream(s4 + i + 768);
        __stcs(d4 + i, a); __stcs(d4 + i + 256, b); __stcs(d4 + i + 512, c); __stcs(d4 + i + 768, d);
      }
      for (; i < nv; i += 256) __stcs(d4 + i, ldg_stream(s4 + i));
    } else {
      for (int64_t i = threadIdx.x; i < nbytes; i += 256) dp[i] = sp[i];
    }
  }
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
  kv_round_kernel<<<unsigned((state->n_slots + kKvWarps - 1) / kKvWarps), kKvWarps * 32, 0, st>>>(
      *policy, *state, *kv);
  if (kv->kv_pool) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t slots = int64_t(state->n_slots) * policy->max_branches;
    const unsigned grid = unsigned(slots < 4 * sms ? slots : 4 * sms);
    kv_copy_kernel<<<grid, 256, 0, st>>>(*kv, state->n_slots, policy->max_branches);
  }
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
