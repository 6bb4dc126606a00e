// K3 slot update (kv_round_kernel, kv.cu; see there for the design).
#pragma once
#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kKvWarps = 4;
constexpr int kArTop = 0, kArHwm = 1, kArOwner = 2, kArPeak = 3;
constexpr int kWin = 16;         // entries per lane per window (512 per warp)
constexpr int kForkWin = 8;      // fork-copy entries per lane per window (256 per warp)

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
        if (i < nv) d4[i] = v[u];          // write-back stores (as K3's C4 copies)
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
// Optional phase timestamps (DuchessState.trace, words 16-19 of the slot's
// record: start, after the forks, after the releases, end).
__device__ __forceinline__ void kv_trace(const DuchessState& s, int r, int k, int lane) {
  if (s.trace && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    s.trace[int64_t(r) * DUCHESS_TRACE_WORDS + k] = (long long)t;
  }
}

// The update of slot r (one warp; `ws` = kv_warp_words(B) shared words of
// this warp).
static __device__ __noinline__ void kv_slot_round(const DuchessPolicy& pol, const DuchessState& s,
                                           const DuchessKV& kv, int r, int lane, int32_t* ws) {
  kv_trace(s, r, 16, lane);
  const int B = s.branch_cap, C = pol.max_branches, NB = kv.max_blocks, bt = kv.block_tokens;
  const int P = kv.blocks_per_slot;
  int32_t* bk = ws;                                                // [B] tokens covered
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
    if (nf <= 32) {
      // All forks at once. Their roots are branches alive before this round
      // (never a child of it) and the children's rows are distinct, so the
      // row copies are independent: the (fork, block) entries are flattened
      // and copied a window at a time. The tail blocks are popped in record
      // order: the k-th tail-needing fork takes stk[top - 1 - k], then fresh
      // blocks above the high-water mark.
      const bool fv = lane < nf && bs[fc] == DUCHESS_ACTIVE;     // cancelled / ended at once
      const int nfull = fv ? fp / bt : 0;
      const int tl = fv ? fp - nfull * bt : 0;
      int tot;
      const int off = warp_excl_scan(nfull, lane, tot);
      if (lane < nf) bo[lane] = off;
      const unsigned tmask = __ballot_sync(0xffffffffu, tl > 0);
      const int trank = __popc(tmask & ((1u << lane) - 1u));
      const int ntail = __popc(tmask);
      int tblk = -1, tsrc = -1;
      if (tl > 0) {
        if (trank < top) tblk = stk[top - 1 - trank];
        else if (hwm + (trank - top) < P) tblk = hwm + (trank - top);
        tsrc = row(fr_)[nfull];                                   // the root's partial block
      }
      if (fv) bk[fc] = fp;
      __syncwarp();
      for (int w0 = 0; w0 < tot; w0 += kForkWin * 32) {
        int v[kForkWin], dch[kForkWin], dj[kForkWin];
#pragma unroll
        for (int u = 0; u < kForkWin; ++u) {
          const int e = w0 + u * 32 + lane;
          int lo = 0, hi = nf - 1;                                // last fork with bo <= e
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (bo[mid] <= e) lo = mid; else hi = mid - 1;
          }
          const int root_e = __shfl_sync(0xffffffffu, fr_, lo);
          dch[u] = __shfl_sync(0xffffffffu, fc, lo);
          dj[u] = e - bo[lo];
          v[u] = e < tot ? row(root_e)[dj[u]] : -2;
        }
#pragma unroll
        for (int u = 0; u < kForkWin; ++u) {
          if (v[u] == -2) continue;
          row(dch[u])[dj[u]] = v[u];
          if (v[u] >= 0) atomicAdd(ref + (v[u] - base), 1);      // distinct within a row
        }
      }
      const int from_stack = min(ntail, top);
      const int fresh = min(ntail - from_stack, P - hwm);
      overflow += ntail - from_stack - fresh;
      n_alloc += from_stack + fresh;
      n_jobs = from_stack + fresh;                                // allocated tails: ranks 0..n-1
      top -= from_stack;
      hwm += fresh;
      long long tb = tblk >= 0 ? (long long)(tl) * kv.kv_bytes_per_token : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tb += __shfl_xor_sync(0xffffffffu, tb, o);
      tail_bytes += tb;
      if (tl > 0) {
        row(fc)[nfull] = tblk < 0 ? -1 : tblk + base;
        if (tblk >= 0) {
          ref[tblk] = 1;
          int32_t* jb = jobs + trank * 4;
          jb[0] = tsrc;
          jb[1] = tblk + base;
          jb[2] = tl;
        }
      }
      if (kv.kv_pool) {
        // copy the partial tails' KV bytes (warp-wide 16-byte streams)
        const int64_t block_bytes = kv.kv_bytes_per_token * bt;
        unsigned m = __ballot_sync(0xffffffffu, tblk >= 0);
        while (m) {
          const int f = __ffs(m) - 1;
          m &= m - 1;
          const int sb = __shfl_sync(0xffffffffu, tsrc, f);
          const int db = __shfl_sync(0xffffffffu, tblk, f);
          const int tt = __shfl_sync(0xffffffffu, tl, f);
          kv_copy_bytes(kv.kv_pool + int64_t(sb) * block_bytes,
                        kv.kv_pool + int64_t(db + base) * block_bytes,
                        int64_t(tt) * kv.kv_bytes_per_token, lane);
        }
      }
      __syncwarp();
    } else {
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
    }
    kv_trace(s, r, 17, lane);
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

  kv_trace(s, r, 18, lane);
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
  kv_trace(s, r, 19, lane);
  __syncwarp();
}

}  // namespace duchess
