// K2: per-request orchestration decisions, one warp per request slot.
//
// Restates DuchessRun.step (reference pkg/src/branchsim/orchestrator.py:329-402)
// for every request slot at once, bit-exact:
//   duchess_advance: refill finished slots from the service queue
//                    (RequestRun.__init__ seeding, :242-248) then phase 1,
//                    decode chunk + natural-end / cap collection (:344-355).
//   [K1 scores the survivors' activation windows between the two launches]
//   duchess_decide : phase 2 predictions (:357-363), phase 3 early termination
//                    (:365-373), phase 4 branch-out refill (:375-388), phase 5
//                    request termination + majority vote (:390-399).
//
// IEEE fidelity: this translation unit is compiled with --fmad=false and uses
// explicit _rn intrinsics wherever the reference's double arithmetic could
// otherwise be contracted; random draws replay CPython's MT19937
// genrand_res53; the branch-out normaliser replays CPython >= 3.12's
// compensated (Neumaier) builtin sum().
#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "score_core.cuh"
#include "../../include/duchess_b200.h"

namespace cg = cooperative_groups;

namespace duchess {

#ifndef DUCHESS_K2_WARPS
#define DUCHESS_K2_WARPS 4
#endif
constexpr int kWarpsPerBlock = DUCHESS_K2_WARPS;
constexpr int kMaxC = DUCHESS_MAX_SLOTS;
constexpr int kMtN = 624, kMtM = 397;
// DuchessState.active_count words: [0], [1] survivor rows listed per parity,
// [2] parity of the list the next scorer launch reads, [3] unused (zero),
// [4..5] duchess_round's 64-bit accumulator (rows listed | slots out << 32).
enum : int { kListPar = 2, kListAcc = 4 };
constexpr double kProbFloor = 1e-6;   // orchestrator.py:56 BRANCH_PROB_FLOOR

// ---------------------------------------------------------------------------
// MT19937, CPython flavour (Modules/_randommodule.c genrand_uint32 / random()).

__device__ __forceinline__ uint32_t mt_temper(uint32_t y) {
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

__device__ __forceinline__ uint32_t mt_mix(uint32_t a, uint32_t b, uint32_t m) {
  const uint32_t y = (a & 0x80000000u) | (b & 0x7fffffffu);
  return m ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
}

// Regenerate all 624 words, warp-cooperatively. The serial recurrence splits
// into phases whose members only read words finalised by earlier phases.
__device__ void mt_twist_warp(uint32_t* mt, int lane) {
  auto phase = [&](int lo, int hi, bool old_m) {
    for (int base = lo; base < hi; base += 32) {
      const int kk = base + lane;
      uint32_t nv = 0;
      const bool act = kk < hi;
      if (act) {
        const uint32_t m = old_m ? mt[kk + kMtM] : mt[kk + kMtM - kMtN];
        nv = mt_mix(mt[kk], mt[kk + 1], m);
      }
      __syncwarp();
      if (act) mt[kk] = nv;
      __syncwarp();
    }
  };
  phase(0, kMtN - kMtM, true);               // [0, 227): mt[kk+397] still old
  phase(kMtN - kMtM, 2 * (kMtN - kMtM), false);  // [227, 454): mt[kk-227] from phase A
  phase(2 * (kMtN - kMtM), kMtN - 1, false);     // [454, 623): mt[kk-227] from phase B
  if (lane == 0) mt[kMtN - 1] = mt_mix(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
  __syncwarp();
}

// Produce n tempered words into out[] (shared), advancing the stream.
__device__ void mt_words_warp(uint32_t* mt, int n, uint32_t* out, int lane) {
  int idx = int(mt[kMtN]);
  int k = 0;
  while (k < n) {
    if (idx >= kMtN) {
      mt_twist_warp(mt, lane);
      idx = 0;
    }
    const int take = min(n - k, kMtN - idx);
    for (int j = lane; j < take; j += 32) out[k + j] = mt_temper(mt[idx + j]);
    k += take;
    idx += take;
  }
  __syncwarp();
  if (lane == 0) mt[kMtN] = uint32_t(idx);
  __syncwarp();
}

// random.random(): (a*67108864.0 + b) * (1.0/9007199254740992.0), exact.
__device__ __forceinline__ double mt_res53(uint32_t w0, uint32_t w1) {
  const double a = double(w0 >> 5), b = double(w1 >> 6);
  return __dmul_rn(__dadd_rn(__dmul_rn(a, 67108864.0), b), 1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------------------
// Template lookups (workload.py:82-106).

__device__ __forceinline__ int upper_bound(const int32_t* a, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// probe_answer (workload.py:82-94). Answer id 0 is NO_ANSWER ("").
__device__ __forceinline__ int probe_answer(const DuchessWorkload& w, int t, int pos) {
  const int conv = w.conv[t];
  if (conv >= 0 && pos >= conv) return w.final_ans[t];
  const int lo = w.probe_off[t], hi = w.probe_off[t + 1];
  if (hi > lo) {
    const int idx = upper_bound(w.probe_at, lo, hi, pos) - 1;
    if (idx >= lo) return w.probe_ans[idx];
  }
  return 0;
}

// Same lookup with independent loads per level: conv / CSR bounds / final in
// one round trip, then an 8-ary search over probe_at (8 loads per level).
// Invariant: probe_at[i] <= pos for i in [L, lo), probe_at[i] > pos for i in [hi, H).
__device__ __forceinline__ int probe_answer_fast(const DuchessWorkload& w, int t, int pos) {
  const int conv = w.conv[t];
  const int L = w.probe_off[t];
  const int H = w.probe_off[t + 1];
  const int fin = w.final_ans[t];
  if (conv >= 0 && pos >= conv) return fin;
  int lo = L, hi = H;
  while (hi - lo > 8) {
    const int span = hi - lo;
    int idx[8], at[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) idx[q] = lo + (span * (q + 1)) / 9;
#pragma unroll
    for (int q = 0; q < 8; ++q) at[q] = w.probe_at[idx[q]];
    int nlo = lo, nhi = hi;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (at[q] <= pos) nlo = idx[q] + 1;
      else nhi = min(nhi, idx[q]);
    }
    lo = nlo;
    hi = nhi;
  }
  int at8[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) at8[q] = (lo + q < hi) ? w.probe_at[lo + q] : 0x7fffffff;
  int k = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) k += at8[q] <= pos;
  const int ans = lo + k - 1;
  return ans >= L ? w.probe_ans[ans] : 0;
}

// probe_answer_fast with the template's (conv, probe CSR bounds, final)
// already in registers: only the search levels touch memory.
__device__ __forceinline__ int probe_answer_pref(const DuchessWorkload& w, int conv, int L, int H,
                                                 int fin, int pos) {
  if (conv >= 0 && pos >= conv) return fin;
  int lo = L, hi = H;
  while (hi - lo > 8) {
    const int span = hi - lo;
    int idx[8], at[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) idx[q] = lo + (span * (q + 1)) / 9;
#pragma unroll
    for (int q = 0; q < 8; ++q) at[q] = w.probe_at[idx[q]];
    int nlo = lo, nhi = hi;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (at[q] <= pos) nlo = idx[q] + 1;
      else nhi = min(nhi, idx[q]);
    }
    lo = nlo;
    hi = nhi;
  }
  int at8[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) at8[q] = (lo + q < hi) ? w.probe_at[lo + q] : 0x7fffffff;
  int k = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) k += at8[q] <= pos;
  const int ans = lo + k - 1;
  return ans >= L ? w.probe_ans[ans] : 0;
}

// trace_prediction (workload.py:97-106).
__device__ __forceinline__ double trace_prediction(const DuchessWorkload& w, int t, int pos) {
  const int lo = w.pred_off[t], hi = w.pred_off[t + 1];
  if (hi <= lo) return 0.0;
  const int idx = upper_bound(w.pred_at, lo, hi, pos) - 1;
  return idx < lo ? 0.0 : w.pred_p[idx];
}

// min(max(p, 1e-6), 1.0) ** exponent (orchestrator.py:183).
__device__ __forceinline__ double branch_raw(double p, double inv_temp) {
  const double x = fmin(fmax(p, kProbFloor), 1.0);
  if (inv_temp == 1.0 || x == 1.0) return x;
  return pow(x, inv_temp);
}

// CPython >= 3.12 builtin sum() over floats: Neumaier compensation.
struct NeumaierSum {
  double f = 0.0, c = 0.0;
  __device__ __forceinline__ void add(double x) {
    const double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
    f = t;
  }
  __device__ __forceinline__ double result() const {
    return (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f;
  }
};

// branch_out_sample (orchestrator.py:188-197) given precomputed raws and
// their compensated sum; flags draws within 4 ulp of a CDF boundary.
__device__ int sample_index(const double* raw, int n, double total, double u, bool* ambiguous) {
  double acc = 0.0, prev = 0.0;
  int pick = n - 1;
  for (int j = 0; j < n; ++j) {
    const double w = __ddiv_rn(raw[j], total);
    prev = acc;
    acc = __dadd_rn(acc, w);
    if (u < acc) { pick = j; break; }
  }
  const double tol = 4.0 * 2.220446049250313e-16;
  *ambiguous = fabs(u - acc) <= tol * fmax(acc, 1e-300) ||
               (pick > 0 && fabs(u - prev) <= tol * fmax(prev, 1e-300));
  return pick;
}

// Sequential CDF walk over precomputed weights (orchestrator.py:192-197).
__device__ __forceinline__ int cdf_pick(const double* w, int n, double u, bool* ambiguous) {
  double acc = 0.0, prev = 0.0;
  int pick = n - 1;
  for (int j = 0; j < n; ++j) {
    prev = acc;
    acc = __dadd_rn(acc, w[j]);
    if (u < acc) { pick = j; break; }
  }
  const double tol = 4.0 * 2.220446049250313e-16;
  *ambiguous = fabs(u - acc) <= tol * fmax(acc, 1e-300) ||
               (pick > 0 && fabs(u - prev) <= tol * fmax(prev, 1e-300));
  return pick;
}

// ---------------------------------------------------------------------------
// Per-warp shared-memory cache of one request slot. Active branches are exactly
// the occupied branch slots (a slot is released whenever its branch leaves
// ACTIVE), so a round only touches <= C branches: they are gathered once with
// independent loads, processed in shared memory, and every state change is
// stored straight back (stores are off the critical path).

struct SlotCache {
  int bid[kMaxC];        // branch id occupying slot j, -1 = free
  int off[kMaxC], dec[kMaxC], streak[kMaxC], status[kMaxC], npred[kMaxC];
  double lp[kMaxC];
  int rank[kMaxC];       // creation-order rank of slot j among occupied slots
  int order[kMaxC];      // occupied slots in creation (branch id) order
  int need[kMaxC];       // survivor needs a synthetic draw
  int free_slots[kMaxC];
  int nat_child[kMaxC];
  int alive_slot[kMaxC];
  int alive_root[kMaxC];
  int src_idx[kMaxC];
  double raw[kMaxC];
  double raw_slot[kMaxC];  // branch_raw of slot j's new prediction (phase 2)
  double wts[kMaxC];
  double draws[kMaxC];
  int nat[kMaxC];        // natural length of the template in slot j (for phase 1)
  int t0, n_tmpl, rounds, tok_dec, tok_prb;   // request's template base / count, counters
  int need_refill;                    // set by decide_slot: the request just finished
  int tally_delta[64];   // this round's terminations, per answer id (answer_cap <= 64)
  uint32_t words[2 * kMaxC];
  uint32_t mt[kMtN + 1];
};

__device__ __forceinline__ int warp_count_flags(const int32_t* flags, int upto, int lane) {
  int cnt = 0;
  for (int base = 0; base < upto; base += 128) {
    int f[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = base + q * 32 + lane;
      f[q] = j < upto ? flags[j] : 0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) cnt += __popc(__ballot_sync(0xffffffffu, f[q] != 0));
  }
  return cnt;
}

__device__ __forceinline__ void load_slot(const DuchessState& s, int64_t rC, int64_t rB, int C,
                                          SlotCache& c, int lane) {
  for (int j = lane; j < C; j += 32) {
    const int b = s.slot_branch[rC + j];
    c.bid[j] = b;
    if (b >= 0) {
      const int64_t bi = rB + b;
      c.off[j] = s.br_offset[bi];
      c.dec[j] = s.br_decoded[bi];
      c.streak[j] = s.br_streak[bi];
      c.status[j] = s.br_status[bi];
      c.npred[j] = s.br_npred[bi];
      c.lp[j] = s.br_last_pred[bi];
    }
  }
  __syncwarp();
}

// Per-request fields phase 1 needs (template base, counters, the occupied
// slots' template lengths) when the slot cache was not filled by decide_slot.
__device__ __forceinline__ void load_meta(const DuchessWorkload& w, const DuchessState& s, int r,
                                          int p, int C, SlotCache& c, int lane) {
  const int t0 = w.tmpl_off[p];
  const int t1 = w.tmpl_off[p + 1];
  if (lane == 0) {
    c.t0 = t0;
    c.n_tmpl = t1 - t0;
    c.rounds = s.rounds[r];
    c.tok_dec = s.tokens_decode[r];
    c.tok_prb = s.tokens_probe[r];
  }
  for (int j = lane; j < C; j += 32)
    if (c.bid[j] >= 0) c.nat[j] = w.nat_len[t0 + c.bid[j]];
  __syncwarp();
}

// Creation-order ranks of occupied slots; returns the number occupied.
// Branch ids are unique within a request, so with C <= 32 and ids < 256 a
// slot's rank is a popcount over a warp-wide OR of id bits (one redux per 32
// ids, all independent) instead of a serial scan of the C slots.
__device__ __forceinline__ int order_slots(SlotCache& c, int C, int B, int lane) {
  if (C <= 32 && B <= 256) {
    const int b = lane < C ? c.bid[lane] : -1;
    const bool occ = b >= 0;
    const int bw = b >> 5;
    const unsigned bit = 1u << (b & 31);
    int rk = 0, n = 0;
    const int nw = (B + 31) >> 5;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q >= nw) break;
      const unsigned m = __reduce_or_sync(0xffffffffu, occ && bw == q ? bit : 0u);
      const int pc = __popc(m);
      rk += bw > q ? pc : (bw == q ? __popc(m & (bit - 1u)) : 0);
      n += pc;
    }
    if (occ) {
      c.rank[lane] = rk;
      c.order[rk] = lane;
    }
    __syncwarp();
    return n;
  }
  int n = 0;
  for (int base = 0; base < C; base += 32) {
    const int j = base + lane;
    const bool occ = j < C && c.bid[j] >= 0;
    if (occ) {
      const int b = c.bid[j];
      int rk = 0;
      for (int k = 0; k < C; ++k) rk += (c.bid[k] >= 0 && c.bid[k] < b);
      c.rank[j] = rk;
      c.order[rk] = j;
    }
    n += __popc(__ballot_sync(0xffffffffu, occ));
  }
  __syncwarp();
  return n;
}

constexpr int kMtPerLane = (kMtN + 1 + 31) / 32;   // 20

// Batched copy of the 625-word state: all loads issued before any store.
__device__ __forceinline__ void copy_mt(const uint32_t* src, uint32_t* dst, int lane) {
  uint32_t v[kMtPerLane];
#pragma unroll
  for (int q = 0; q < kMtPerLane; ++q) {
    const int j = q * 32 + lane;
    v[q] = j <= kMtN ? src[j] : 0u;
  }
#pragma unroll
  for (int q = 0; q < kMtPerLane; ++q) {
    const int j = q * 32 + lane;
    if (j <= kMtN) dst[j] = v[q];
  }
  __syncwarp();
}

// Slot MT states are copy-on-write: a refill stores only the index word with
// kMtPristine set, and the words are read from the pool's initial state
// (DuchessWorkload.mt_init[p], which the host stores already twisted, index
// 0) until the first twist writes a private copy. So a refill copies nothing
// and a fresh request's first draws need no twist.
constexpr uint32_t kMtPristine = 0x80000000u;

// n tempered words from a global-memory stream whose words live at `src`
// (mt_g itself, or the pool's initial state while `flag` == kMtPristine).
// Common case (no twist due): read src[idx, idx+n) and bump the index.
// Otherwise stage the state in shared memory, run the warp-parallel twist
// there, and write the (now private) state back to mt_g.
__device__ int mt_words_global(uint32_t* mt_g, const uint32_t*& src, uint32_t& flag,
                               uint32_t* mt_s, int idx, int n, uint32_t* out, int lane) {
  if (idx + n <= kMtN) {
    for (int k = lane; k < n; k += 32) out[k] = mt_temper(src[idx + k]);
    __syncwarp();
    if (lane == 0) mt_g[kMtN] = uint32_t(idx + n) | flag;
    __syncwarp();
    return idx + n;
  }
  copy_mt(src, mt_s, lane);
  if (lane == 0) mt_s[kMtN] = uint32_t(idx);
  __syncwarp();
  mt_words_warp(mt_s, n, out, lane);
  const int nidx = int(mt_s[kMtN]);
  copy_mt(mt_s, mt_g, lane);
  src = mt_g;
  flag = 0u;
  return nidx;
}

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Refill slot r with pool request p: RequestRun.__init__ (:242-248).
// `qr` (optional): the queue position's record (pool index, template base,
// template count, MT index word), one 16-byte load instead of three.
__device__ void refill_slot(const DuchessPolicy& pol, const DuchessWorkload& w,
                            const DuchessState& s, int r, int p, SlotCache& c, int lane,
                            const int4* qr = nullptr) {
  const int C = pol.max_branches;
  const int64_t rC = int64_t(r) * C, rB = int64_t(r) * s.branch_cap;
  const int t0 = qr ? qr->y : w.tmpl_off[p];
  const int n_tmpl = qr ? qr->z : w.tmpl_off[p + 1] - t0;
  const int seeded = min(C, n_tmpl);
  for (int j = lane; j < C; j += 32) {
    const bool live = j < seeded;
    if (live) c.nat[j] = w.nat_len[t0 + j];
    c.bid[j] = live ? j : -1;
    c.off[j] = 0; c.dec[j] = 0; c.streak[j] = 0; c.status[j] = DUCHESS_ACTIVE;
    c.npred[j] = 0; c.lp[j] = 0.5;
    s.slot_branch[rC + j] = live ? j : -1;
    if (live) {
      const int64_t bi = rB + j;
      s.br_offset[bi] = 0; s.br_decoded[bi] = 0; s.br_streak[bi] = 0;
      s.br_status[bi] = DUCHESS_ACTIVE; s.br_final[bi] = -1; s.br_npred[bi] = 0;
      s.br_slot[bi] = j; s.br_last_pred[bi] = 0.5;
      if (s.br_probe_last) { s.br_probe_last[bi] = -1; s.br_probe_run[bi] = 0; }
    }
  }
  for (int a = lane; a < s.answer_cap; a += 32) s.tally[int64_t(r) * s.answer_cap + a] = 0;
  if (lane == 0) {
    s.mt[int64_t(r) * DUCHESS_MT_WORDS + kMtN] =
        kMtPristine | (qr ? uint32_t(qr->w) : w.mt_init[int64_t(p) * DUCHESS_MT_WORDS + kMtN]);
    s.slot_req[r] = p;
    if (s.slot_aux) s.slot_aux[r] = 0;
    s.n_branches[r] = seeded;
    s.next_template[r] = seeded;
    s.tokens_decode[r] = 0;
    s.tokens_probe[r] = 0;
    s.rounds[r] = 0;
    s.done[r] = 0;
    c.t0 = t0;
    c.n_tmpl = n_tmpl;
    c.rounds = 0;
    c.tok_dec = 0;
    c.tok_prb = 0;
  }
  __syncwarp();
}

// Optional per-slot phase timestamps (DuchessState.trace, 8 x int64 per slot).
__device__ __forceinline__ void trace_mark(const DuchessState& s, int r, int k, int lane) {
  if (s.trace && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    s.trace[int64_t(r) * DUCHESS_TRACE_WORDS + k] = (long long)t;
  }
}

// Phase-1 record of the round in flight: round, decoding, max_chunk,
// decode_tokens, probes, pool request (round 0 = no round started).
constexpr int kP1Words = 8;

// Refill-or-load prologue of a round (RequestRun.__init__ on refill).
// Returns the pool request in slot r, or -1 if the slot stays idle.
__device__ int slot_prologue(const DuchessPolicy& pol, const DuchessWorkload& w,
                             const DuchessState& s, int r, SlotCache& c, int lane,
                             bool cache_valid) {
  const int C = pol.max_branches;
  const int64_t rC = int64_t(r) * C, rB = int64_t(r) * s.branch_cap;
  // the k-th slot needing a refill (slot order) takes queue[head + k]
  const int head = s.queue_head[0];
  if (r == 0) {
    const int total = warp_count_flags(s.needs_refill, s.n_slots, lane);
    const int avail = w.cycle ? total : max(0, min(total, w.queue_len - head));
    if (lane == 0) s.queue_head[1] = head + avail;
  }
  if (s.needs_refill[r]) {
    const int q = head + warp_count_flags(s.needs_refill, r, lane);
    int p = -1;
    if (w.queue_len > 0) {
      if (w.cycle) p = w.queue[q % w.queue_len];
      else if (q < w.queue_len) p = w.queue[q];
    }
    if (p < 0) {
      if (lane == 0) { s.slot_req[r] = -1; s.done[r] = 1; }
      __syncwarp();
      return -1;
    }
    refill_slot(pol, w, s, r, p, c, lane);
    return p;
  }
  if (s.done[r]) return -1;
  const int p = s.slot_req[r];
  if (p < 0) return -1;
  if (!cache_valid) {
    load_slot(s, rC, rB, C, c, lane);
    load_meta(w, s, r, p, C, c, lane);
  }
  return p;
}

// Survivor list phase 1 appends to (the round kernel writes the next round's
// list parity while the scorer reads the current one).
struct Phase1Out {
  int32_t* rows;
  int32_t* count;
  bool defer;            // do not append: report the survivor masks instead
  unsigned mask[2];      // (defer) survivor branch slots, 32 per word
};

__device__ void phase1_slot(const DuchessPolicy& pol, const DuchessWorkload& w,
                            const DuchessState& s, int r, int p, SlotCache& c, int lane,
                            Phase1Out* fo = nullptr) {
  int32_t* list_rows = fo ? fo->rows : s.active_rows;
  int32_t* list_count = fo ? fo->count : s.active_count;
  if (!fo && s.active_rows) {                      // split launches: the current parity
    const int par = s.active_count[kListPar];
    list_rows += int64_t(par) * s.n_slots * pol.max_branches;
    list_count += par;
  }
  int n_listed = 0;
  const int C = pol.max_branches;
  const int64_t rC = int64_t(r) * C, rB = int64_t(r) * s.branch_cap;
  int32_t* p1 = s.p1_rec + int64_t(r) * kP1Words;
  // ---- phase 1: decode one interval per active branch (:344-355) ----
  const int t0 = c.t0;
  int decoding = 0, max_chunk = 0, dtok = 0, probes = 0;
  for (int base = 0; base < C; base += 32) {
    const int j = base + lane;
    const int b = j < C ? c.bid[j] : -1;
    bool surv = false;
    if (b >= 0) {
      const int64_t bi = rB + b;
      const int t = t0 + b;                           // branch_id == template_index (:260-266)
      const int nat = c.nat[j];
      int pos = c.off[j] + c.dec[j];
      const int room = min(nat, pol.token_cap) - pos;            // _decode_chunk :273-279
      const int chunk = max(0, min(pol.interval_tokens, room));
      c.dec[j] += chunk;
      pos += chunk;
      if (chunk > 0) { decoding++; max_chunk = max(max_chunk, chunk); dtok += chunk; }
      s.br_decoded[bi] = c.dec[j];
      int ans = -1, status = DUCHESS_ACTIVE;
      if (pos >= nat) { ans = w.final_ans[t]; status = DUCHESS_NATURAL_END; }
      else if (pos >= pol.token_cap) { ans = probe_answer_fast(w, t, pos); status = DUCHESS_CAPPED; probes++; }
      if (status != DUCHESS_ACTIVE) {                 // _collect (:287-290), slot released
        s.br_status[bi] = status;
        s.br_final[bi] = ans;
        s.br_slot[bi] = -1;
        atomicAdd(&s.tally[int64_t(r) * s.answer_cap + ans], 1);
        s.slot_branch[rC + j] = -1;
      } else {
        surv = true;
        s.row_mask[rC + j] = 1;
        s.row_pos[rC + j] = pos;
        s.row_tmpl[rC + j] = b;
        s.row_req[rC + j] = p;
      }
    }
    // compacted list of windows for the persistent scorer (order irrelevant)
    const unsigned m = __ballot_sync(0xffffffffu, surv);
    n_listed += __popc(m);
    if (fo && fo->defer) {
      fo->mask[base >> 5] = m;
    } else if (m && list_rows) {
      int basei = 0;
      if (lane == 0) basei = atomicAdd(list_count, __popc(m));
      basei = __shfl_sync(0xffffffffu, basei, 0);
      if (surv) list_rows[basei + __popc(m & ((1u << lane) - 1u))] = int32_t(rC + j);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    decoding += __shfl_xor_sync(0xffffffffu, decoding, o);
    dtok += __shfl_xor_sync(0xffffffffu, dtok, o);
    probes += __shfl_xor_sync(0xffffffffu, probes, o);
    max_chunk = max(max_chunk, __shfl_xor_sync(0xffffffffu, max_chunk, o));
  }
  if (lane == 0) {
    const int rounds = c.rounds + 1;
    c.rounds = rounds;
    c.tok_dec += dtok;
    c.tok_prb += probes * pol.probe_cost_tokens;
    s.rounds[r] = rounds;
    s.tokens_decode[r] = c.tok_dec;
    s.tokens_probe[r] = c.tok_prb;
    p1[0] = rounds;
    p1[1] = decoding;
    p1[2] = max_chunk;
    p1[3] = dtok;
    p1[4] = probes;
    p1[5] = p;
    p1[6] = t0;                  // template base / count: the decision of this
    p1[7] = c.n_tmpl;            // round gathers the template headers in wave 2
  }
}

__device__ void clear_round_inputs(const DuchessPolicy& pol, const DuchessState& s, int r, int lane) {
  const int C = pol.max_branches;
  for (int j = lane; j < C; j += 32) s.row_mask[int64_t(r) * C + j] = 0;
  if (lane < kP1Words) s.p1_rec[int64_t(r) * kP1Words + lane] = 0;
  __syncwarp();
}

// Queue records a round's refills will most likely take: lane i holds the
// record at queue position head + i, head = the pop counter read when the
// round starts (pops happen late in the round; a position outside the window,
// e.g. after a stale head, is loaded when popped). Read in the decision's
// gather waves, so it overlaps the scorer's tail.
struct QueuePrefetch {
  int head;
  int4 rec;
};

__device__ __forceinline__ void prefetch_queue_rec(const DuchessWorkload& w, QueuePrefetch& qp,
                                                   int lane) {
  qp.rec = make_int4(-1, 0, 0, 0);
  if (w.queue_rec && w.queue_len > 0) {
    const int q = qp.head + lane;
    if (w.cycle || q < w.queue_len)
      qp.rec = __ldg(reinterpret_cast<const int4*>(w.queue_rec) + (w.cycle ? q % w.queue_len : q));
  }
}

// Phases 2-5 for slot r whose phase-1 record is live (cache not yet loaded
// unless cache_loaded). Completes round_rec. Returns the pool request decided.
__device__ int decide_slot(const DuchessPolicy& pol, const DuchessWorkload& w,
                            const DuchessState& s, int r, SlotCache& c, int lane,
                            const double* probs, bool wait_inputs = false,
                            QueuePrefetch* qp = nullptr) {
  const int C = pol.max_branches;
  const int64_t rC = int64_t(r) * C, rB = int64_t(r) * s.branch_cap;
  const int64_t rA = int64_t(r) * s.answer_cap;
  int32_t* rec = s.round_rec + int64_t(r) * DUCHESS_REC_WORDS;
  const int32_t* p1 = s.p1_rec + int64_t(r) * kP1Words;
  uint32_t* mt_g = s.mt + int64_t(r) * DUCHESS_MT_WORDS;
  int32_t* act = s.actions + int64_t(r) * 2 * C * 3;
  const bool dev_probs = pol.pred_source != DUCHESS_PRED_TRACE;
  const bool small_tally = s.answer_cap <= 64;
  trace_mark(s, r, 0, lane);
  // Waves 1-3 read only state finished by the previous round and read-only
  // tables, never the scorer's output, so under programmatic dependent
  // launch (wait_inputs) they run before griddepcontrol.wait, overlapping
  // the scorer's tail; mutable state is read through L2 (ld.cg).
  // ---- wave 1: everything addressed by the slot alone, issued together ----
  const int p1v = lane < kP1Words ? __ldcg(p1 + lane) : 0;
  const int sb0 = lane < C ? __ldcg(s.slot_branch + rC + lane) : -1;
  const int sb1 = lane + 32 < C ? __ldcg(s.slot_branch + rC + lane + 32) : -1;
  int tl0 = 0, tl1 = 0;
  if (small_tally) {
    if (lane < s.answer_cap) tl0 = __ldcg(s.tally + rA + lane);
    if (lane + 32 < s.answer_cap) tl1 = __ldcg(s.tally + rA + lane + 32);
  }
  const uint32_t mt_iw = __ldcg(mt_g + kMtN);
  if (qp) qp->head = __ldcg(s.queue_head + 1);
  uint32_t mt_flag = mt_iw & kMtPristine;
  int mt_idx = int(mt_iw & ~kMtPristine);
  const int nb = __ldcg(s.n_branches + r);
  const int next_t = __ldcg(s.next_template + r);
  const int cnt_dec = __ldcg(s.tokens_decode + r), cnt_prb = __ldcg(s.tokens_probe + r);
  const int cnt_rnd = __ldcg(s.rounds + r);
  const int p = __shfl_sync(0xffffffffu, p1v, 5);
  if (lane < DUCHESS_REC_WORDS) {
    const int v = __shfl_sync(0x00000fffu, p1v, lane < DUCHESS_REC_NACTIONS ? lane : 5);
    rec[lane] = lane < DUCHESS_REC_NACTIONS ? v : (lane == DUCHESS_REC_REQ ? v : 0);
  }
  if (lane < 64) c.tally_delta[lane] = 0;
  c.tally_delta[lane + 32 < 64 ? lane + 32 : 63] = 0;
  // template base / count, recorded by phase 1 (no dependent tmpl_off load)
  const int t0 = __shfl_sync(0xffffffffu, p1v, 6);
  const int n_tmpl = __shfl_sync(0xffffffffu, p1v, 7);
  // ---- wave 2: branch fields, template headers (below) ----
  const uint32_t* mt_src = mt_flag ? w.mt_init + int64_t(p) * DUCHESS_MT_WORDS : mt_g;
  c.bid[lane] = -1;
  if (lane + 32 < kMaxC) c.bid[lane + 32] = -1;
  {
    const int sbs[2] = {sb0, sb1};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = lane + 32 * q;
      const int b = sbs[q];
      if (j < C) c.bid[j] = b;
      if (b >= 0) {
        const int64_t bi = rB + b;
        c.off[j] = __ldcg(s.br_offset + bi);
        c.dec[j] = __ldcg(s.br_decoded + bi);
        c.streak[j] = __ldcg(s.br_streak + bi);
        c.status[j] = __ldcg(s.br_status + bi);
        c.npred[j] = __ldcg(s.br_npred + bi);
        c.lp[j] = __ldcg(s.br_last_pred + bi);
      }
    }
  }
  // ---- wave 3: per-survivor template headers (speculative: used only if the
  // branch terminates), child template lengths, MT words a round can consume ----
  int hconv[2], hlo[2], hhi[2], hfin[2];
  {
    const int sbs[2] = {sb0, sb1};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      hconv[q] = -1; hlo[q] = 0; hhi[q] = 0; hfin[q] = 0;
      if (sbs[q] >= 0) {
        const int t = t0 + sbs[q];
        hconv[q] = w.conv[t];
        hlo[q] = w.probe_off[t];
        hhi[q] = w.probe_off[t + 1];
        hfin[q] = w.final_ans[t];
      }
    }
  }
  for (int k = lane; k < C && next_t + k < n_tmpl; k += 32)
    c.nat_child[k] = w.nat_len[t0 + next_t + k];      // templates a fork could consume
  if (sb0 >= 0) c.nat[lane] = w.nat_len[t0 + sb0];     // next round's phase 1
  if (sb1 >= 0) c.nat[lane + 32] = w.nat_len[t0 + sb1];
  if (lane == 0) { c.t0 = t0; c.n_tmpl = n_tmpl; }
  const bool words_ready = dev_probs && mt_idx + 2 * C <= kMtN;
  if (words_ready)
    for (int k = lane; k < 2 * C; k += 32) c.words[k] = mt_temper(__ldcg(mt_src + mt_idx + k));
  // Each survivor's CoT-probe answer at its position (probe_answer,
  // workload.py:82-94), searched now — speculatively, before the scorer's
  // results are needed — for the branch that terminates this round and for
  // the synthetic predictor's oracle term.
  int pans[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if ((q == 0 ? sb0 : sb1) >= 0)
      pans[q] = probe_answer_pref(w, hconv[q], hlo[q], hhi[q], hfin[q], c.off[j] + c.dec[j]);
  }
  __syncwarp();
  const int n_surv = order_slots(c, C, s.branch_cap, lane);
  if (qp) prefetch_queue_rec(w, *qp, lane);
  // Probabilities from the device probe (fp32 logits, within 1e-4 *
  // max(|logit|, 1) of the fp64 reference, BASELINE.json north_star): count
  // the predictions close enough to tau that an fp64 probe could have put
  // them on the other side of `p > tau` (expected rare).
  double band_lo = 2.0, band_hi = -1.0;
  if (pol.pred_source == DUCHESS_PRED_DEVICE && pol.early_term_threshold > 0.0 && pol.early_term_threshold < 1.0) {
    const double lt = log(pol.early_term_threshold / (1.0 - pol.early_term_threshold));
    const double tol = 1e-4 * fmax(fabs(lt), 1.0);
    band_lo = 1.0 / (1.0 + exp(-(lt - tol)));
    band_hi = 1.0 / (1.0 + exp(-(lt + tol)));
  }
  if (wait_inputs) pdl_wait();                     // the scorer's probabilities are final
  double pr0 = 0.0, pr1 = 0.0;
  if (dev_probs) {
    if (lane < C) pr0 = __ldcg(probs + (rC + lane) * pol.n_layers);
    if (lane + 32 < C) pr1 = __ldcg(probs + (rC + lane + 32) * pol.n_layers);
  }
  trace_mark(s, r, 1, lane);

  // ---- phase 2: predictions, creation order (:357-363) ----
  int n_need = 0;
  if (pol.pred_source == DUCHESS_PRED_TRACE) {
    for (int base = 0; base < C; base += 32) {
      const int j = base + lane;
      bool nd = false;
      if (j < C && c.bid[j] >= 0) {
        const int t = t0 + c.bid[j];
        nd = w.pred_off[t + 1] <= w.pred_off[t];
        c.need[j] = nd;
      }
      n_need += __popc(__ballot_sync(0xffffffffu, nd));
    }
    __syncwarp();
    if (n_need > 0) {
      mt_idx = mt_words_global(mt_g, mt_src, mt_flag, c.mt, mt_idx, 2 * n_need, c.words, lane);
      for (int k = lane; k < n_need; k += 32) c.draws[k] = mt_res53(c.words[2 * k], c.words[2 * k + 1]);
      __syncwarp();
    }
  }
  const double tau = pol.early_term_threshold;
  int n_term = 0;
  int n_near_tau = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    const int b = j < C ? c.bid[j] : -1;
    bool term = false;
    if (b >= 0) {
      const int64_t bi = rB + b;
      const int t = t0 + b;
      const int pos = c.off[j] + c.dec[j];
      double pr;
      if (pol.pred_source == DUCHESS_PRED_TRACE) {
        if (!c.need[j]) {
          pr = trace_prediction(w, t, pos);
        } else {
          int k = 0;                                     // rank among draw-needing survivors
          for (int qq = 0; qq < C; ++qq) k += (c.bid[qq] >= 0 && c.bid[qq] < b && c.need[qq]);
          const double u = c.draws[k];
          // synthetic_predict (predictor.py:328-335) on probe_answer == ground truth
          const int pa = pans[q];
          const double oracle = pa == w.ground_truth[p] ? 1.0 : 0.0;
          const double v = __dadd_rn(__dmul_rn(pol.rho, oracle), __dmul_rn(__dsub_rn(1.0, pol.rho), u));
          pr = fmin(fmax(v, 0.0), 1.0);
        }
      } else if (pol.pred_source == DUCHESS_PRED_HOST || pol.n_layers == 1 || pol.combine == 0) {
        pr = q == 0 ? pr0 : pr1;
      } else {
        double acc = 0.0;
        for (int l = 0; l < pol.n_layers; ++l) acc = __dadd_rn(acc, __ldcg(probs + (rC + j) * pol.n_layers + l));
        pr = __ddiv_rn(acc, double(pol.n_layers));
      }
      n_near_tau += pr > band_lo && pr < band_hi;
      const int streak = pr > tau ? c.streak[j] + 1 : 0;   // strict > (:363)
      c.lp[j] = pr;
      // branch-out weight of this prediction (:183), computed here so its pow
      // overlaps the phase-3 stores; read back for the branches still alive
      c.raw_slot[j] = branch_raw(pr, pol.inv_temperature);
      c.npred[j] += 1;
      c.streak[j] = streak;
      s.step_pred[rC + j] = pr;
      s.br_last_pred[bi] = pr;
      s.br_npred[bi] = c.npred[j];
      s.br_streak[bi] = streak;
      // ---- phase 3: early termination (:365-373) ----
      term = streak >= pol.early_term_rounds;
      const int k = c.rank[j];
      act[k * 3 + 0] = term ? DUCHESS_ACT_TERMINATE : DUCHESS_ACT_CONTINUE;
      act[k * 3 + 1] = b;
      act[k * 3 + 2] = -1;
      if (term) {
        const int ans = pans[q];
        c.status[j] = DUCHESS_EARLY_TERMINATED;
        s.br_status[bi] = DUCHESS_EARLY_TERMINATED;
        s.br_final[bi] = ans;
        s.br_slot[bi] = -1;
        atomicAdd(&s.tally[rA + ans], 1);
        if (small_tally) atomicAdd(&c.tally_delta[ans], 1);
      }
    }
    n_term += __popc(__ballot_sync(0xffffffffu, term));
  }
  if (pol.pred_source == DUCHESS_PRED_DEVICE) {
    n_near_tau = __reduce_add_sync(0xffffffffu, n_near_tau);
    if (lane == 0 && n_near_tau) add_counter(&s.counters[DUCHESS_CNT_NEAR_TAU], n_near_tau);
  }
  __syncwarp();

  trace_mark(s, r, 2, lane);
  // ---- phase 4: branch-out refill of freed slots (:375-388) ----
  // alive = survivors still ACTIVE in creation order; entry j is held in
  // registers by lane j % 32 (set j / 32, C <= 64). Free slots ascending.
  int n_alive = 0, n_free = 0;
  for (int base = 0; base < C; base += 32) {
    const int i = base + lane;
    bool alive = false;
    int j = -1;
    if (i < n_surv) {
      j = c.order[i];
      alive = c.status[j] == DUCHESS_ACTIVE;
    }
    const unsigned am = __ballot_sync(0xffffffffu, alive);
    if (alive) c.alive_slot[n_alive + __popc(am & ((1u << lane) - 1u))] = j;
    n_alive += __popc(am);
    const int sj = base + lane;
    const bool fr = sj < C && (c.bid[sj] < 0 || c.status[sj] != DUCHESS_ACTIVE);
    const unsigned fm = __ballot_sync(0xffffffffu, fr);
    if (fr) c.free_slots[n_free + __popc(fm & ((1u << lane) - 1u))] = sj;
    n_free += __popc(fm);
  }
  __syncwarp();
  int sl0 = -1, sl1 = -1, rt0 = -1, rt1 = -1, ps0 = 0, ps1 = 0;
  double lp0 = 0.0, lp1 = 0.0, rw0 = 0.0, rw1 = 0.0;
  if (lane < n_alive) {
    sl0 = c.alive_slot[lane]; rt0 = c.bid[sl0]; ps0 = c.off[sl0] + c.dec[sl0]; lp0 = c.lp[sl0];
    rw0 = c.raw_slot[sl0];
    c.raw[lane] = rw0;
  }
  if (lane + 32 < n_alive) {
    sl1 = c.alive_slot[lane + 32]; rt1 = c.bid[sl1]; ps1 = c.off[sl1] + c.dec[sl1]; lp1 = c.lp[sl1];
    rw1 = c.raw_slot[sl1];
    c.raw[lane + 32] = rw1;
  }
  const int n_forks = n_alive > 0 ? max(0, min(C - n_alive, n_tmpl - next_t)) : 0;
  __syncwarp();
  trace_mark(s, r, 3, lane);
  if (n_forks > 0) {
    if (words_ready) {                                 // words prefetched in wave 3
      if (lane == 0) mt_g[kMtN] = uint32_t(mt_idx + 2 * n_forks) | mt_flag;
      mt_idx += 2 * n_forks;
    } else {
      mt_idx = mt_words_global(mt_g, mt_src, mt_flag, c.mt, mt_idx, 2 * n_forks, c.words, lane);
    }
    // Tree-order prefix sums of the raws, extended by one entry per fork.
    double P0 = warp_incl_scan(rw0, lane);
    double P1 = warp_incl_scan(rw1, lane) + __shfl_sync(0xffffffffu, P0, 31);
    // u of fork k, held by lane k % 32 (set k / 32), all drawn up front
    double u0 = 0.0, u1 = 0.0;
    if (lane < n_forks) u0 = mt_res53(c.words[2 * lane], c.words[2 * lane + 1]);
    if (lane + 32 < n_forks) u1 = mt_res53(c.words[2 * lane + 64], c.words[2 * lane + 65]);
    // The serial part: fork k picks entry idx_k of the list alive + children
    // 0..k-1 (each child repeats its source's raw); lane k % 32 records idx_k.
    // Child fields are resolved after the loop.
    trace_mark(s, r, 20, lane);
    int pick0 = -1, pick1 = -1, n = n_alive, amb = 0;
    // Tree prefix of the last entry, tracked in a register: each child's prefix
    // is p_last + raw, the same sum the appending lane stores. It is also the
    // normaliser of the fast path: the reference's is CPython's compensated
    // sum() (:184), which the fast path needs only to within a few ulp (a sum
    // of n positive terms in any order is within (n - 1) ulp of the exact
    // total; the margin below absorbs that), and the exact compensated sum is
    // replayed from the raws (creation order) only on the rare fallback.
    double p_last = __shfl_sync(0xffffffffu, (n - 1) >= 32 ? P1 : P0, (n - 1) & 31);
    // margin factor 4 (2n + 9) ulp, stepped by 8 ulp per appended entry
    constexpr double kUlp4 = 4.0 * 1.1102230246251565e-16;
    double mfac = double(2 * n + 9) * kUlp4;
    for (int k = 0; k < n_forks; ++k) {
      const double u = __shfl_sync(0xffffffffu, k < 32 ? u0 : u1, k & 31);
      // The reference picks the first j with u < acc_j, acc_j the sequential
      // sum of fl(raw_i / total_c). acc_j, P_j / total and the running sum
      // differ by less than (3n + 10) ulp of the total, so away from a
      // 4 (2n + 9) ulp margin the pick is read off the prefixes; otherwise
      // lane 0 replays the exact sequential walk with the compensated total.
      const double thr = __dmul_rn(u, p_last);
      const double margin = mfac * p_last;
      const bool v0 = lane < n, v1 = lane + 32 < n;
      const bool near = (v0 && fabs(thr - P0) <= margin) || (v1 && fabs(thr - P1) <= margin);
      // the prefix-sum pick and the margin vote side by side (no branch between)
      const unsigned b0 = __ballot_sync(0xffffffffu, v0 && thr < P0);
      const unsigned b1 = __ballot_sync(0xffffffffu, v1 && thr < P1);
      const bool any_near = __any_sync(0xffffffffu, near);
      int idx = b0 ? __ffs(b0) - 1 : (b1 ? 32 + __ffs(b1) - 1 : n - 1);
      if ((pol.flags & DUCHESS_FLAG_EXACT_CDF) || any_near) {
        __syncwarp();                                       // c.raw[0, n) written
        NeumaierSum sum;
        for (int q = 0; q < n; ++q) sum.add(c.raw[q]);
        const double total = sum.result();
        if (v0) c.wts[lane] = __ddiv_rn(rw0, total);
        if (v1) c.wts[lane + 32] = __ddiv_rn(rw1, total);
        __syncwarp();
        idx = 0;
        if (lane == 0) {
          bool ambiguous = false;
          idx = cdf_pick(c.wts, n, u, &ambiguous);
          amb += ambiguous;
        }
        idx = __shfl_sync(0xffffffffu, idx, 0);
      }
      const double src_raw = __shfl_sync(0xffffffffu, idx >= 32 ? rw1 : rw0, idx & 31);
      p_last = __dadd_rn(p_last, src_raw);
      if (lane == (n & 31)) {                               // append child k as entry n
        if (n < 32) { rw0 = src_raw; P0 = p_last; }
        else        { rw1 = src_raw; P1 = p_last; }
      }
      if (lane == (k & 31)) {
        if (k < 32) pick0 = idx; else pick1 = idx;
      }
      if (lane == 0) c.raw[n] = src_raw;                    // for the exact fallback
      mfac += 2.0 * kUlp4;
      ++n;
    }
    __syncwarp();
    trace_mark(s, r, 21, lane);
    // Resolve children by pointer jumping over the pick chains: a child's
    // source is an alive entry or an earlier child. Root / last_prediction
    // come from the alive entry at the chain's end; the offset is the
    // source's position clamped by each child's template length along the
    // chain (_spawn clamp, :263).
    {
      const int na = n_alive;
      int ptr0 = pick0, ptr1 = pick1;
      int m0 = lane < n_forks ? c.nat_child[lane] : 0x7fffffff;
      int m1 = lane + 32 < n_forks ? c.nat_child[lane + 32] : 0x7fffffff;
      // value of entry j held as (v0, v1) by lane j % 32 (set j / 32); j is
      // per-lane, so both sets are shuffled and the reader selects
      auto fetch_i = [&](int v0, int v1, int j) {
        const int a = __shfl_sync(0xffffffffu, v0, j & 31);
        const int b = __shfl_sync(0xffffffffu, v1, j & 31);
        return j >= 32 ? b : a;
      };
      auto fetch_d = [&](double v0, double v1, int j) {
        const double a = __shfl_sync(0xffffffffu, v0, j & 31);
        const double b = __shfl_sync(0xffffffffu, v1, j & 31);
        return j >= 32 ? b : a;
      };
      const int C_hi = n_forks > 32;                         // any child in set 1
#pragma unroll 1
      for (int it = 0; (1 << it) < n_forks; ++it) {
        const int q0 = ptr0 >= na ? ptr0 - na : 0, q1 = ptr1 >= na ? ptr1 - na : 0;
        const int pj0 = fetch_i(ptr0, ptr1, q0), mj0 = fetch_i(m0, m1, q0);
        int pj1 = 0, mj1 = 0;
        if (C_hi) { pj1 = fetch_i(ptr0, ptr1, q1); mj1 = fetch_i(m0, m1, q1); }
        if (lane < n_forks && ptr0 >= na) { m0 = min(m0, mj0); ptr0 = pj0; }
        if (lane + 32 < n_forks && ptr1 >= na) { m1 = min(m1, mj1); ptr1 = pj1; }
      }
      // ptr now names an alive entry: fetch its slot / root / position / lp
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = lane + 32 * q;
        const int ptr = q == 0 ? ptr0 : ptr1;
        const int pick = q == 0 ? pick0 : pick1;
        const int mm = q == 0 ? m0 : m1;
        if (q == 1 && !C_hi) break;
        const int e = max(ptr, 0);
        const int a_root = fetch_i(rt0, rt1, e);
        const int a_pos = fetch_i(ps0, ps1, e);
        const double a_lp = fetch_d(lp0, lp1, e);
        if (k < n_forks) {
          const int child_slot = c.free_slots[k];
          c.nat[child_slot] = c.nat_child[k];
          c.bid[child_slot] = nb + k;
          c.off[child_slot] = min(a_pos, mm);
          c.dec[child_slot] = 0;
          c.streak[child_slot] = 0;
          c.status[child_slot] = DUCHESS_ACTIVE;
          c.npred[child_slot] = 0;
          c.lp[child_slot] = a_lp;                         // inherits last_prediction (:264)
          // source: an alive entry's slot, or the slot of an earlier child
          c.src_idx[k] = pick < na ? -1 - c.alive_slot[pick] : pick - na;
          c.alive_root[k] = a_root;
        }
      }
      __syncwarp();
    }
    trace_mark(s, r, 22, lane);
    if (lane == 0) {
      if (amb) add_counter(&s.counters[DUCHESS_CNT_AMBIGUOUS], (long long)(amb));
      add_counter(&s.counters[DUCHESS_CNT_FORKS], (long long)(n_forks));
      s.n_branches[r] = nb + n_forks;
      s.next_template[r] = next_t + n_forks;
    }
    __syncwarp();
    for (int k = lane; k < n_forks; k += 32) {
      const int cs = c.free_slots[k];
      const int child = nb + k;
      const int si = c.src_idx[k];
      const int src = si < 0 ? c.bid[-1 - si] : nb + si;   // source branch id
      const int64_t ci = rB + child;
      s.br_offset[ci] = c.off[cs];
      s.br_decoded[ci] = 0;
      s.br_streak[ci] = 0;
      s.br_status[ci] = DUCHESS_ACTIVE;
      s.br_final[ci] = -1;
      s.br_npred[ci] = 0;
      s.br_last_pred[ci] = c.lp[cs];
      s.br_slot[ci] = cs;
      const int a = n_surv + k;
      act[a * 3 + 0] = DUCHESS_ACT_BRANCH_OUT;
      act[a * 3 + 1] = child;
      act[a * 3 + 2] = src;
      int32_t* f = s.forks + (rC + k) * 4;
      f[0] = child;
      f[1] = src;
      f[2] = c.alive_root[k];
      f[3] = c.off[cs];
    }
  }
  __syncwarp();

  trace_mark(s, r, 4, lane);
  // ---- phase 5: request termination (:390-399) ----
  int max_count = 0, total = 0, best = 0x7fffffff;
  int cnt0 = 0, cnt1 = 0;
  if (small_tally) {                 // tally prefetched in wave 1 + this round's terminations
    if (lane < s.answer_cap) cnt0 = tl0 + c.tally_delta[lane];
    if (lane + 32 < s.answer_cap) cnt1 = tl1 + c.tally_delta[lane + 32];
    total = cnt0 + cnt1;
    if (cnt0 > 0) { max_count = cnt0; best = lane; }
    if (cnt1 > max_count) { max_count = cnt1; best = lane + 32; }
  } else {
    for (int a = lane; a < s.answer_cap; a += 32) {
      const int cnt = __ldcg(&s.tally[rA + a]);
      total += cnt;
      if (cnt > max_count) { max_count = cnt; best = a; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    total += __shfl_xor_sync(0xffffffffu, total, o);
    const int mc = __shfl_xor_sync(0xffffffffu, max_count, o);
    const int bb = __shfl_xor_sync(0xffffffffu, best, o);
    if (mc > max_count || (mc == max_count && bb < best)) { max_count = mc; best = bb; }
  }
  int reason = DUCHESS_REASON_NONE;
  if (max_count >= pol.need_consensus) reason = DUCHESS_REASON_CONSENSUS;
  else if (total >= pol.need_coverage) reason = DUCHESS_REASON_COVERAGE;
  bool any_active = false;
  for (int base = 0; base < C; base += 32) {
    const int j = base + lane;
    bool a = j < C && c.bid[j] >= 0 && c.status[j] == DUCHESS_ACTIVE;
    if (a && reason != DUCHESS_REASON_NONE) {        // _cancel_active (:292-294)
      s.br_status[rB + c.bid[j]] = DUCHESS_CANCELLED;
      s.br_slot[rB + c.bid[j]] = -1;
      c.bid[j] = -1;
    }
    if (j < C && (c.bid[j] < 0 || c.status[j] != DUCHESS_ACTIVE)) c.bid[j] = -1;
    if (j < C) s.slot_branch[rC + j] = c.bid[j];
    any_active |= __any_sync(0xffffffffu, a);
  }
  if (reason == DUCHESS_REASON_NONE && !any_active) reason = DUCHESS_REASON_EXHAUSTED;
  const bool done = reason != DUCHESS_REASON_NONE;
  trace_mark(s, r, 5, lane);
  if (s.trace && lane == 0) { s.trace[int64_t(r) * DUCHESS_TRACE_WORDS + 6] = n_forks; s.trace[int64_t(r) * DUCHESS_TRACE_WORDS + 7] = n_term; }
  if (done) {
    if (small_tally) {
      if (lane < s.answer_cap) s.out_tally[int64_t(p) * s.answer_cap + lane] = cnt0;
      if (lane + 32 < s.answer_cap) s.out_tally[int64_t(p) * s.answer_cap + lane + 32] = cnt1;
    } else {
      for (int a = lane; a < s.answer_cap; a += 32)
        s.out_tally[int64_t(p) * s.answer_cap + a] = __ldcg(&s.tally[rA + a]);
    }
  }
  if (lane == 0) {
    c.need_refill = done ? 1 : 0;
    c.rounds = cnt_rnd;
    c.tok_dec = cnt_dec;
    c.tok_prb = cnt_prb + n_term * pol.probe_cost_tokens;
    s.tokens_probe[r] = c.tok_prb;
    rec[DUCHESS_REC_PROBES] = p1[4] + n_term;
    rec[DUCHESS_REC_NACTIONS] = n_surv + n_forks;
    rec[DUCHESS_REC_NFORKS] = n_forks;
    rec[DUCHESS_REC_NSURV] = n_surv;
    rec[DUCHESS_REC_DONE] = done ? 1 : 0;
    add_counter(&s.counters[DUCHESS_CNT_BRANCH_STEPS], (long long)(n_surv));
    if (done) {
      const bool empty = total == 0;   // majority_vote on an empty tally raises (core.py:80-81)
      s.done[r] = 1;
      s.needs_refill[r] = 1;
      rec[DUCHESS_REC_REASON] = reason;
      rec[DUCHESS_REC_FINAL] = empty ? -1 : best;
      s.out_final[p] = empty ? -1 : best;
      s.out_reason[p] = reason;
      s.out_tokens_decode[p] = c.tok_dec;
      s.out_tokens_probe[p] = c.tok_prb;
      s.out_rounds[p] = c.rounds;
      s.out_error[p] = empty ? 1 : 0;
      add_counter(&s.counters[DUCHESS_CNT_FINISHED], 1ll);
      if (empty) add_counter(&s.counters[DUCHESS_CNT_ERRORS], 1ll);
    } else {
      s.needs_refill[r] = 0;
    }
  }
  return p;
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
advance_kernel(DuchessPolicy pol, DuchessWorkload w, DuchessState s) {
  __shared__ SlotCache cache[kWarpsPerBlock];
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= s.n_slots) return;
  SlotCache& c = cache[threadIdx.x >> 5];
  clear_round_inputs(pol, s, r, lane);
  const int p = slot_prologue(pol, w, s, r, c, lane, false);
  if (p >= 0) phase1_slot(pol, w, s, r, p, c, lane);
}

__device__ __forceinline__ void decide_prologue(const DuchessState& s) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.queue_head[0] = s.queue_head[1];
    if (s.active_count) s.active_count[s.active_count[kListPar]] = 0;   // consumed by the scorer
  }
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
decide_kernel(DuchessPolicy pol, DuchessWorkload w, DuchessState s, const double* probs) {
  __shared__ SlotCache cache[kWarpsPerBlock];
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  decide_prologue(s);
  if (r >= s.n_slots) return;
  if (s.p1_rec[int64_t(r) * kP1Words] == 0) {     // slot idle or finished: no round
    if (lane == 0) s.round_rec[int64_t(r) * DUCHESS_REC_WORDS + DUCHESS_REC_ROUND] = 0;
    return;
  }
  decide_slot(pol, w, s, r, cache[threadIdx.x >> 5], lane, probs);
}

// Refill-or-load prologue with the service queue popped atomically in
// completion order (the round kernel has no grid-wide barrier to rank slots).
__device__ int slot_prologue_atomic(const DuchessPolicy& pol, const DuchessWorkload& w,
                                   const DuchessState& s, int r, SlotCache& c, int lane,
                                   bool cache_valid, int32_t* pop, int p_decided = -1,
                                   const QueuePrefetch* qp = nullptr) {
  const int C = pol.max_branches;
  if (cache_valid ? c.need_refill : s.needs_refill[r]) {
    int q = 0;
    if (lane == 0) q = atomicAdd(pop, 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    int p = -1;
    int4 rec;
    const int4* qr = nullptr;
    if (w.queue_len > 0 && (w.cycle || q < w.queue_len)) {
      const int qi = w.cycle ? q % w.queue_len : q;
      if (w.queue_rec) {
        const int d = qp ? q - qp->head : -1;
        if (d >= 0 && d < 32) {                        // prefetched at kernel start
          rec.x = __shfl_sync(0xffffffffu, qp->rec.x, d);
          rec.y = __shfl_sync(0xffffffffu, qp->rec.y, d);
          rec.z = __shfl_sync(0xffffffffu, qp->rec.z, d);
          rec.w = __shfl_sync(0xffffffffu, qp->rec.w, d);
        } else {
          rec = reinterpret_cast<const int4*>(w.queue_rec)[qi];
        }
        p = rec.x;
        qr = &rec;
      } else {
        p = w.queue[qi];
      }
    }
    if (p < 0) {
      if (lane == 0) { s.slot_req[r] = -1; s.done[r] = 1; s.needs_refill[r] = 0; }
      __syncwarp();
      return -1;
    }
    refill_slot(pol, w, s, r, p, c, lane, qr);
    if (lane == 0) s.needs_refill[r] = 0;
    __syncwarp();
    return p;
  }
  // decided this round and not finished: still serving the same request
  if (cache_valid && p_decided >= 0) return p_decided;
  if (s.done[r]) return -1;
  const int p = s.slot_req[r];
  if (p < 0) return -1;
  if (!cache_valid) {
    load_slot(s, int64_t(r) * C, int64_t(r) * s.branch_cap, C, c, lane);
    load_meta(w, s, r, p, C, c, lane);
  }
  return p;
}

// Round boundary: decide round k, then refill + phase 1 of round k+1, per
// slot with no grid-wide barrier: a finished slot pops the service queue
// atomically (the requests admitted per round are the same as with ranked
// refills; only their slot placement follows completion order), and phase 1
// appends the slot's survivors to the other parity's list. The last warp
// resets the consumed list and flips the parity.
// Two warps per CTA: small enough (18 KB shared) to become resident next to
// the scorer's CTAs, which trigger this launch early (programmatic dependent
// launch), so each slot's state prefetch overlaps the scorer's tail.
constexpr int kRoundWarps = 2;

__global__ void __maxnreg__(128)
round_kernel(DuchessPolicy pol, DuchessWorkload w, DuchessState s, const double* probs) {
  __shared__ SlotCache cache[kRoundWarps];
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kRoundWarps + (threadIdx.x >> 5);
  SlotCache& c = cache[threadIdx.x >> 5];
  if (r >= s.n_slots) return;
  trace_mark(s, r, 12, lane);
  const bool had_round = __ldcg(s.p1_rec + int64_t(r) * kP1Words) != 0;
  QueuePrefetch qp;
  int p_dec = -1;
  if (had_round) {
    p_dec = decide_slot(pol, w, s, r, c, lane, probs, true, &qp);   // waits for the scorer
  } else {
    qp.head = __ldcg(s.queue_head + 1);
    prefetch_queue_rec(w, qp, lane);
    pdl_wait();
    if (lane == 0) s.round_rec[int64_t(r) * DUCHESS_REC_WORDS + DUCHESS_REC_ROUND] = 0;
  }
  const int par = s.active_count[kListPar];
  trace_mark(s, r, 8, lane);
  clear_round_inputs(pol, s, r, lane);
  const int p = slot_prologue_atomic(pol, w, s, r, c, lane, had_round, s.queue_head + 1,
                                     p_dec, &qp);
  trace_mark(s, r, 10, lane);
  Phase1Out fo{};
  fo.defer = true;
  if (p >= 0) phase1_slot(pol, w, s, r, p, c, lane, &fo);
  trace_mark(s, r, 11, lane);
  // One 64-bit atomic per slot both reserves the slot's run of the next list
  // (low word: rows listed so far) and counts the slot out (high word): the
  // last warp out publishes the count and flips the list parity. No fence
  // before it: everything this warp wrote is read only after the kernel
  // boundary, and its queue pop (a returning atomic, consumed above) was
  // performed before this one was issued; the last warp reads the pop counter
  // with an atomic, at L2.
  const int n0 = __popc(fo.mask[0]), n1 = __popc(fo.mask[1]);
  unsigned long long old = 0;
  if (lane == 0)
    old = atomicAdd(reinterpret_cast<unsigned long long*>(s.active_count + kListAcc),
                    (1ull << 32) | unsigned(n0 + n1));
  old = __shfl_sync(0xffffffffu, old, 0);
  const int base = int(uint32_t(old));
  int32_t* rows = s.active_rows + int64_t(par ^ 1) * s.n_slots * pol.max_branches;
  const int64_t rC = int64_t(r) * pol.max_branches;
  const unsigned below = (1u << lane) - 1u;
  if (fo.mask[0] >> lane & 1u) rows[base + __popc(fo.mask[0] & below)] = int32_t(rC + lane);
  if (fo.mask[1] >> lane & 1u) rows[base + n0 + __popc(fo.mask[1] & below)] = int32_t(rC + 32 + lane);
  if (lane == 0 && int(old >> 32) == s.n_slots - 1) {
    s.active_count[par ^ 1] = base + n0 + n1;    // the list the next scorer reads
    s.active_count[par] = 0;                     // consumed by the scorer this round
    s.active_count[kListPar] = par ^ 1;
    *reinterpret_cast<unsigned long long*>(s.active_count + kListAcc) = 0ull;
    s.queue_head[0] = atomicAdd(s.queue_head + 1, 0);
  }
  trace_mark(s, r, 13, lane);
}

// ---------------------------------------------------------------------------
// Baseline policies (orchestrator.py:405-561) on the same slot machinery.

// _finish (:296-304) for the baselines: tally -> majority vote, outcome record.
__device__ void close_slot(const DuchessState& s, int r, int p, int reason, int lane,
                           int32_t* rec) {
  const int64_t rA = int64_t(r) * s.answer_cap;
  int max_count = 0, total = 0, best = 0x7fffffff;
  for (int a = lane; a < s.answer_cap; a += 32) {
    const int cnt = __ldcg(&s.tally[rA + a]);
    total += cnt;
    if (cnt > max_count) { max_count = cnt; best = a; }
    s.out_tally[int64_t(p) * s.answer_cap + a] = cnt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    total += __shfl_xor_sync(0xffffffffu, total, o);
    const int mc = __shfl_xor_sync(0xffffffffu, max_count, o);
    const int bb = __shfl_xor_sync(0xffffffffu, best, o);
    if (mc > max_count || (mc == max_count && bb < best)) { max_count = mc; best = bb; }
  }
  if (lane == 0) {
    const bool empty = total == 0;
    s.done[r] = 1;
    s.needs_refill[r] = 1;
    rec[DUCHESS_REC_DONE] = 1;
    rec[DUCHESS_REC_REASON] = reason;
    rec[DUCHESS_REC_FINAL] = empty ? -1 : best;
    s.out_final[p] = empty ? -1 : best;
    s.out_reason[p] = reason;
    s.out_tokens_decode[p] = s.tokens_decode[r];
    s.out_tokens_probe[p] = s.tokens_probe[r];
    s.out_rounds[p] = s.rounds[r];
    s.out_error[p] = empty ? 1 : 0;
    add_counter(&s.counters[DUCHESS_CNT_FINISHED], 1ll);
    if (empty) add_counter(&s.counters[DUCHESS_CNT_ERRORS], 1ll);
  }
}

__device__ void baseline_slot(const DuchessPolicy& pol, const DuchessWorkload& w,
                              const DuchessState& s, int r, int p, SlotCache& c, int lane) {
  const int C = pol.max_branches;
  const int64_t rC = int64_t(r) * C, rB = int64_t(r) * s.branch_cap;
  const int64_t rA = int64_t(r) * s.answer_cap;
  int32_t* rec = s.round_rec + int64_t(r) * DUCHESS_REC_WORDS;
  int32_t* act = s.actions + int64_t(r) * 2 * C * 3;
  const int t0 = w.tmpl_off[p];
  const int n_tmpl = w.tmpl_off[p + 1] - t0;
  const int kind = pol.policy_kind;
  // ShortMk bookkeeping (:454-455): m finishers end the request
  const int target = min(pol.short_m, min(C, n_tmpl));
  const int finished0 = (kind == DUCHESS_POLICY_SHORT_MK) ? s.slot_aux[r] : 0;
  // per-slot plan in registers (slots j = lane, lane + 32)
  int chunk[2] = {0, 0}, pos0[2] = {0, 0}, nat[2] = {0, 0}, tt[2] = {0, 0};
  bool occ[2] = {false, false}, fin[2] = {false, false};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if (j < C && c.bid[j] >= 0) {
      occ[q] = true;
      tt[q] = t0 + c.bid[j];
      nat[q] = w.nat_len[tt[q]];
      pos0[q] = c.off[j] + c.dec[j];
      const int room = min(nat[q], pol.token_cap) - pos0[q];
      chunk[q] = kind == DUCHESS_POLICY_SHORT_MK ? min(pol.interval_tokens, room)
                                                  : max(0, min(pol.interval_tokens, room));
      fin[q] = kind == DUCHESS_POLICY_SHORT_MK && chunk[q] == room;
    }
  }
  // ShortMk: finishers ordered by (chunk, branch id); cut at the m-th (:480-484)
  int cut = -1, n_fin = 0;
  if (kind == DUCHESS_POLICY_SHORT_MK) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = lane + 32 * q;
      if (j < C) c.need[j] = fin[q] ? chunk[q] : -1;      // reuse: finisher chunk or -1
      n_fin += __popc(__ballot_sync(0xffffffffu, fin[q]));
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = lane + 32 * q;
      if (fin[q]) {
        int rk = 0;
        for (int k = 0; k < C; ++k) {
          const int ck = c.need[k];
          if (ck >= 0 && (ck < chunk[q] || (ck == chunk[q] && c.bid[k] < c.bid[j]))) ++rk;
        }
        c.rank[j] = rk;
        c.order[rk] = chunk[q];
      }
    }
    __syncwarp();
    if (finished0 + n_fin >= target) cut = c.order[target - finished0 - 1];
  }
  int decoding = 0, max_chunk = 0, dtok = 0, probes = 0, counted = 0;
  bool cont[2] = {false, false};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if (!occ[q]) continue;
    const int b = c.bid[j];
    const int64_t bi = rB + b;
    const int take = (kind == DUCHESS_POLICY_SHORT_MK && cut >= 0) ? min(chunk[q], cut) : chunk[q];
    const int pos = pos0[q] + take;
    c.dec[j] += take;
    s.br_decoded[bi] = c.dec[j];
    if (take > 0) { decoding++; max_chunk = max(max_chunk, take); dtok += take; }
    int status = DUCHESS_ACTIVE, ans = -1;
    if (kind == DUCHESS_POLICY_SHORT_MK) {
      // _finish_branch (:457-464) for counted finishers
      const bool collect = fin[q] && (cut < 0 || (c.rank[j] < target - finished0 && chunk[q] <= cut));
      if (collect) {
        counted++;
        if (pos >= nat[q]) { status = DUCHESS_NATURAL_END; ans = w.final_ans[tt[q]]; }
        else { status = DUCHESS_CAPPED; ans = probe_answer_fast(w, tt[q], pos); probes++; }
      }
    } else if (pos >= nat[q]) {
      status = DUCHESS_NATURAL_END; ans = w.final_ans[tt[q]];
    } else if (pos >= pol.token_cap) {
      status = DUCHESS_CAPPED; ans = probe_answer_fast(w, tt[q], pos); probes++;
    } else if (kind == DUCHESS_POLICY_DYNASOR) {
      ans = probe_answer_fast(w, tt[q], pos);                  // probe every round (:553-557)
      probes++;
      const int last = s.br_probe_last[bi];
      const int run = (ans == last) ? s.br_probe_run[bi] + 1 : 1;
      s.br_probe_last[bi] = ans;
      s.br_probe_run[bi] = run;
      if (run >= pol.dynasor_window) status = DUCHESS_EARLY_TERMINATED;
      else ans = -1;
    } else {
      cont[q] = true;                                           // DefaultSc continue (:430-431)
    }
    if (status != DUCHESS_ACTIVE) {
      c.status[j] = status;
      s.br_status[bi] = status;
      s.br_final[bi] = ans;
      s.br_slot[bi] = -1;
      atomicAdd(&s.tally[rA + ans], 1);
      c.bid[j] = -1;
    }
  }
  // continue actions in creation order (branch id == slot for DefaultSc: no forks)
  int n_act = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    const unsigned m = __ballot_sync(0xffffffffu, cont[q]);
    if (cont[q]) {
      const int k = n_act + __popc(m & ((1u << lane) - 1u));
      act[k * 3 + 0] = DUCHESS_ACT_CONTINUE;
      act[k * 3 + 1] = c.bid[j];
      act[k * 3 + 2] = -1;
    }
    n_act += __popc(m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    decoding += __shfl_xor_sync(0xffffffffu, decoding, o);
    dtok += __shfl_xor_sync(0xffffffffu, dtok, o);
    probes += __shfl_xor_sync(0xffffffffu, probes, o);
    counted += __shfl_xor_sync(0xffffffffu, counted, o);
    max_chunk = max(max_chunk, __shfl_xor_sync(0xffffffffu, max_chunk, o));
  }
  __syncwarp();
  bool cancel = kind == DUCHESS_POLICY_SHORT_MK && cut >= 0;
  bool any_active = false;
  for (int base = 0; base < C; base += 32) {
    const int j = base + lane;
    const bool a = j < C && c.bid[j] >= 0;
    if (a && cancel) {                                          // _cancel_active (:292-294)
      s.br_status[rB + c.bid[j]] = DUCHESS_CANCELLED;
      s.br_slot[rB + c.bid[j]] = -1;
      c.bid[j] = -1;
    }
    if (j < C) s.slot_branch[rC + j] = c.bid[j];
    any_active |= __any_sync(0xffffffffu, a && !cancel);
  }
  if (lane == 0) {
    const int rounds = s.rounds[r] + 1;
    s.rounds[r] = rounds;
    s.tokens_decode[r] += dtok;
    s.tokens_probe[r] += probes * pol.probe_cost_tokens;
    if (kind == DUCHESS_POLICY_SHORT_MK) s.slot_aux[r] = cancel ? target : finished0 + counted;
    rec[DUCHESS_REC_ROUND] = rounds;
    rec[DUCHESS_REC_DECODING] = decoding;
    rec[DUCHESS_REC_MAX_CHUNK] = max_chunk;
    rec[DUCHESS_REC_DECODE] = dtok;
    rec[DUCHESS_REC_PROBES] = probes;
    rec[DUCHESS_REC_NACTIONS] = n_act;
    rec[DUCHESS_REC_NFORKS] = 0;
    rec[DUCHESS_REC_NSURV] = 0;
    rec[DUCHESS_REC_DONE] = 0;
    rec[DUCHESS_REC_REQ] = p;
    if (!cancel && any_active) s.needs_refill[r] = 0;
  }
  __syncwarp();
  if (cancel || !any_active) close_slot(s, r, p, DUCHESS_REASON_EXHAUSTED, lane, rec);
}

// One launch per baseline round: each slot's warp refills its slot if the
// request there finished (the service queue popped atomically, so only its
// own flag is read — no ranking over other slots' flags, which this launch
// rewrites), then runs the policy round (which sets / clears the slot's flag
// for the next round). Requests are independent, so which free slot a request
// lands in does not change its outcome. The last warp out (one 64-bit atomic,
// DuchessState.active_count[4..5]) publishes the pop counter to queue_head[0].
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
baseline_round_kernel(DuchessPolicy pol, DuchessWorkload w, DuchessState s) {
  __shared__ SlotCache cache[kWarpsPerBlock];
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= s.n_slots) return;
  int32_t* rec0 = s.round_rec + int64_t(r) * DUCHESS_REC_WORDS;
  if (lane < DUCHESS_REC_WORDS) rec0[lane] = 0;
  __syncwarp();
  SlotCache& c = cache[threadIdx.x >> 5];
  const int p = slot_prologue_atomic(pol, w, s, r, c, lane, /*cache_valid=*/false,
                                     s.queue_head + 1);
  if (p >= 0) baseline_slot(pol, w, s, r, p, c, lane);
  if (lane == 0) {
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(s.active_count + kListAcc);
    if (int(atomicAdd(acc, 1ull << 32) >> 32) == s.n_slots - 1) {
      s.queue_head[0] = atomicAdd(s.queue_head + 1, 0);
      *acc = 0ull;
    }
  }
}

// ---------------------------------------------------------------------------
// Rule primitives, one warp (branch_out_weights / branch_out_sample).
__global__ void branch_out_kernel(const double* probs, int n, double inv_temp, uint32_t* mt,
                                  int n_draws, int32_t* out_idx, double* out_w,
                                  long long* out_amb) {
  extern __shared__ double raw[];
  __shared__ uint32_t words[2 * 256];
  const int lane = threadIdx.x;
  for (int j = lane; j < n; j += 32) raw[j] = branch_raw(probs[j], inv_temp);
  __syncwarp();
  NeumaierSum sum;
  for (int j = 0; j < n; ++j) sum.add(raw[j]);
  const double total = sum.result();
  if (out_w) for (int j = lane; j < n; j += 32) out_w[j] = __ddiv_rn(raw[j], total);
  long long amb = 0;
  for (int base = 0; base < n_draws; base += 256) {
    const int m = min(256, n_draws - base);
    mt_words_warp(mt, 2 * m, words, lane);
    if (lane == 0) {
      for (int k = 0; k < m; ++k) {
        bool a = false;
        out_idx[base + k] = sample_index(raw, n, total, mt_res53(words[2 * k], words[2 * k + 1]), &a);
        amb += a;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && out_amb) *out_amb = amb;
}

// majority_vote + check_request_termination over count vectors.
__global__ void vote_kernel(const int32_t* counts, int n_sets, int n_ans, int need_cons,
                            int need_cov, int32_t* out_final, int32_t* out_reason) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_sets) return;
  const int32_t* c = counts + int64_t(i) * n_ans;
  int best = -1, mc = 0, total = 0;
  for (int a = 0; a < n_ans; ++a) {
    total += c[a];
    if (c[a] > mc) { mc = c[a]; best = a; }
  }
  if (out_final) out_final[i] = total > 0 ? best : -1;
  if (out_reason)
    out_reason[i] = mc >= need_cons ? DUCHESS_REASON_CONSENSUS
                  : total >= need_cov ? DUCHESS_REASON_COVERAGE : DUCHESS_REASON_NONE;
}

__global__ void lookup_kernel(DuchessWorkload w, const int32_t* tmpl, const int32_t* pos, int n,
                              int32_t* out_ans, double* out_pred) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (out_ans) out_ans[i] = probe_answer_fast(w, tmpl[i], pos[i]);
  if (out_pred) out_pred[i] = trace_prediction(w, tmpl[i], pos[i]);
}

// synthetic_predict (predictor.py:328-335) for n calls drawing from one stream.
__global__ void synthetic_kernel(uint32_t* mt, int n, const int32_t* converged, double rho,
                                 double* out) {
  __shared__ uint32_t words[2 * 256];
  const int lane = threadIdx.x;
  for (int base = 0; base < n; base += 256) {
    const int m = min(256, n - base);
    mt_words_warp(mt, 2 * m, words, lane);
    for (int k = lane; k < m; k += 32) {
      const double u = mt_res53(words[2 * k], words[2 * k + 1]);
      const double oracle = converged[base + k] ? 1.0 : 0.0;
      const double v = __dadd_rn(__dmul_rn(rho, oracle), __dmul_rn(__dsub_rn(1.0, rho), u));
      out[base + k] = fmin(fmax(v, 0.0), 1.0);
    }
    __syncwarp();
  }
}

// sample_confused_level (predictor.py:376-386): row-wise CDF walk, one draw per call.
__global__ void confusion_kernel(uint32_t* mt, int n, const int32_t* true_level,
                                 const double* matrix, int32_t* out) {
  __shared__ uint32_t words[2 * 256];
  const int lane = threadIdx.x;
  for (int base = 0; base < n; base += 256) {
    const int m = min(256, n - base);
    mt_words_warp(mt, 2 * m, words, lane);
    if (lane == 0) {
      for (int k = 0; k < m; ++k) {
        const double u = mt_res53(words[2 * k], words[2 * k + 1]);
        const double* row = matrix + (true_level[base + k] - 1) * 5;
        double acc = 0.0;
        int lvl = 5;
        for (int j = 0; j < 5; ++j) {
          acc = __dadd_rn(acc, row[j]);
          if (u < acc) { lvl = j + 1; break; }
        }
        out[base + k] = lvl;
      }
    }
    __syncwarp();
  }
}

// random.Random(seed) for many 64-bit seeds at once (CPython
// Modules/_randommodule.c random_seed -> init_by_array over the seed's 32-bit
// words), then the pending first twist (index 0, as engine.pretwist): one
// warp per state; the seeding recurrences are serial (lane 0), the twist is
// warp-parallel. States [n][625] (words + index).
__global__ void __launch_bounds__(128) mt_seed_kernel(const uint64_t* seeds, int n, uint32_t* out) {
  __shared__ uint32_t sm[4][kMtN + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 4 + warp;
  if (i >= n) return;
  uint32_t* mt = sm[warp];
  if (lane == 0) {
    const uint64_t sd = seeds[i];
    const uint32_t key[2] = {uint32_t(sd), uint32_t(sd >> 32)};
    const int klen = (sd >> 32) ? 2 : 1;
    mt[0] = 19650218u;
    for (int k = 1; k < kMtN; ++k) mt[k] = 1812433253u * (mt[k - 1] ^ (mt[k - 1] >> 30)) + uint32_t(k);
    int a = 1, b = 0;
    for (int k = 0; k < kMtN; ++k) {             // max(N, klen) == N
      mt[a] = (mt[a] ^ ((mt[a - 1] ^ (mt[a - 1] >> 30)) * 1664525u)) + key[b] + uint32_t(b);
      if (++a >= kMtN) { mt[0] = mt[kMtN - 1]; a = 1; }
      if (++b >= klen) b = 0;
    }
    for (int k = 0; k < kMtN - 1; ++k) {
      mt[a] = (mt[a] ^ ((mt[a - 1] ^ (mt[a - 1] >> 30)) * 1566083941u)) - uint32_t(a);
      if (++a >= kMtN) { mt[0] = mt[kMtN - 1]; a = 1; }
    }
    mt[0] = 0x80000000u;
  }
  __syncwarp();
  mt_twist_warp(mt, lane);
  uint32_t* o = out + int64_t(i) * DUCHESS_MT_WORDS;
  for (int k = lane; k < kMtN; k += 32) o[k] = mt[k];
  if (lane == 0) o[kMtN] = 0u;
}

// sample_confused_level for many requests, each with its own fresh stream
// (simengine.py:223-227: rng = random.Random(predict_seeds[order]), one draw).
// States are [n][625] (words + index), pre-twisted by the host (index 0).
__global__ void confusion_streams_kernel(const uint32_t* mt, int n, const int32_t* true_level,
                                         const double* matrix, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* st = mt + int64_t(i) * DUCHESS_MT_WORDS;
  const int idx = int(st[kMtN]);
  const double u = mt_res53(mt_temper(st[idx]), mt_temper(st[idx + 1]));
  const double* row = matrix + (true_level[i] - 1) * 5;
  double acc = 0.0;
  int lvl = 5;
  for (int j = 0; j < 5; ++j) {
    acc = __dadd_rn(acc, row[j]);
    if (u < acc) { lvl = j + 1; break; }
  }
  out[i] = lvl;
}

// Service timeline of run_simulation (simengine.py:247-257) accumulated per
// pool request from the round records: dt = round_time(decoding, max_chunk)
// (when decoding) + probes * probe_cost; the first-token offset is the
// accumulated time after the first round that decoded tokens.
// round_time (simengine.py:51-56): int(round(tokens * (ms_per_token +
// ms_per_extra_branch * (n - 1)))), Python round() = half to even = rint.
__global__ void timeline_kernel(const int32_t* rec, int n_slots, double ms_per_token,
                                double ms_per_extra_branch, long long probe_cost_ms,
                                long long* service_ms, long long* first_token_ms) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_slots) return;
  const int32_t* rr = rec + int64_t(r) * DUCHESS_REC_WORDS;
  if (rr[DUCHESS_REC_ROUND] == 0) return;
  const int p = rr[DUCHESS_REC_REQ];
  const int decoding = rr[DUCHESS_REC_DECODING];
  long long dt = 0;
  if (decoding > 0) {
    const double rate = __dadd_rn(ms_per_token, __dmul_rn(ms_per_extra_branch, double(decoding - 1)));
    dt += (long long)rint(__dmul_rn(double(rr[DUCHESS_REC_MAX_CHUNK]), rate));
  }
  dt += (long long)rr[DUCHESS_REC_PROBES] * probe_cost_ms;
  const long long t = service_ms[p] + dt;
  service_ms[p] = t;
  if (first_token_ms[p] < 0 && rr[DUCHESS_REC_DECODE] > 0) first_token_ms[p] = t;
}

// check_early_termination (orchestrator.py:167-174): last `rounds` strictly > threshold.
__global__ void streak_kernel(const double* hist, const int32_t* off, int n_sets, double thr,
                              int rounds, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_sets) return;
  const int lo = off[i], hi = off[i + 1];
  int ok = hi - lo >= rounds;
  for (int j = hi - rounds; ok && j < hi; ++j) ok = hist[j] > thr;
  out[i] = ok;
}

}  // namespace duchess

using namespace duchess;

static bool state_ok(const DuchessPolicy* pol, const DuchessState* s) {
  return pol && s && pol->max_branches >= 1 && pol->max_branches <= DUCHESS_MAX_SLOTS &&
         s->branch_cap >= 1 && s->answer_cap >= 1 && s->n_slots >= 0;
}

extern "C" int duchess_advance(const DuchessPolicy* policy, const DuchessWorkload* workload,
                               const DuchessState* state, void* stream) {
  if (!state_ok(policy, state) || !workload) return DUCHESS_EINVAL;
  if (state->n_slots == 0) return DUCHESS_OK;
  const unsigned grid = unsigned((state->n_slots + kWarpsPerBlock - 1) / kWarpsPerBlock);
  advance_kernel<<<grid, 32 * kWarpsPerBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      *policy, *workload, *state);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_decide(const DuchessPolicy* policy, const DuchessWorkload* workload,
                              const DuchessState* state, const double* probs, void* stream) {
  if (!state_ok(policy, state) || !workload) return DUCHESS_EINVAL;
  if (policy->pred_source != DUCHESS_PRED_TRACE && probs == nullptr) return DUCHESS_EINVAL;
  if (state->n_slots == 0) return DUCHESS_OK;
  const unsigned grid = unsigned((state->n_slots + kWarpsPerBlock - 1) / kWarpsPerBlock);
  decide_kernel<<<grid, 32 * kWarpsPerBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      *policy, *workload, *state, probs);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_round(const DuchessPolicy* policy, const DuchessWorkload* workload,
                             const DuchessState* state, const double* probs, void* stream) {
  if (!state_ok(policy, state) || !workload) return DUCHESS_EINVAL;
  if (!state->active_rows || !state->active_count) return DUCHESS_EINVAL;
  if (policy->pred_source != DUCHESS_PRED_TRACE && probs == nullptr) return DUCHESS_EINVAL;
  if (state->n_slots == 0) return DUCHESS_OK;
  const unsigned grid = unsigned((state->n_slots + kRoundWarps - 1) / kRoundWarps);
  DuchessPolicy pol = *policy;
  DuchessWorkload w = *workload;
  DuchessState st = *state;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * kRoundWarps);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, round_kernel, pol, w, st, probs);
  return e == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_baseline_round(const DuchessPolicy* policy, const DuchessWorkload* workload,
                                      const DuchessState* state, void* stream) {
  if (!state_ok(policy, state) || !workload) return DUCHESS_EINVAL;
  if (policy->policy_kind < DUCHESS_POLICY_DEFAULT_SC || policy->policy_kind > DUCHESS_POLICY_DYNASOR)
    return DUCHESS_EINVAL;
  if (policy->policy_kind == DUCHESS_POLICY_SHORT_MK && (!state->slot_aux || policy->short_m < 1))
    return DUCHESS_EINVAL;
  if (policy->policy_kind == DUCHESS_POLICY_DYNASOR &&
      (!state->br_probe_last || !state->br_probe_run || policy->dynasor_window < 2))
    return DUCHESS_EINVAL;
  if (state->n_slots == 0) return DUCHESS_OK;
  if (!state->active_count) return DUCHESS_EINVAL;     // the round's exit count
  const unsigned grid = unsigned((state->n_slots + kWarpsPerBlock - 1) / kWarpsPerBlock);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  baseline_round_kernel<<<grid, 32 * kWarpsPerBlock, 0, st>>>(*policy, *workload, *state);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_branch_out_sample(const double* probs, int32_t n, double inv_temperature,
                                         uint32_t* mt_state, int32_t n_draws, int32_t* out_idx,
                                         double* out_weights, long long* out_ambiguous,
                                         void* stream) {
  if (!probs || n < 1 || n > 4096 || n_draws < 0) return DUCHESS_EINVAL;
  if (n_draws > 0 && (!mt_state || !out_idx)) return DUCHESS_EINVAL;
  branch_out_kernel<<<1, 32, size_t(n) * sizeof(double), static_cast<cudaStream_t>(stream)>>>(
      probs, n, inv_temperature, mt_state, n_draws, out_idx, out_weights, out_ambiguous);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_vote(const int32_t* counts, int32_t n_sets, int32_t n_answers,
                            int32_t need_consensus, int32_t need_coverage, int32_t* out_final,
                            int32_t* out_reason, void* stream) {
  if (!counts || n_sets < 0 || n_answers < 0) return DUCHESS_EINVAL;
  if (n_sets == 0) return DUCHESS_OK;
  vote_kernel<<<(n_sets + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, n_sets, n_answers, need_consensus, need_coverage, out_final, out_reason);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_template_lookup(const DuchessWorkload* workload, const int32_t* tmpl,
                                       const int32_t* pos, int32_t n, int32_t* out_probe_answer,
                                       double* out_trace_pred, void* stream) {
  if (!workload || n < 0) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  lookup_kernel<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      *workload, tmpl, pos, n, out_probe_answer, out_trace_pred);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_synthetic_predict(uint32_t* mt_state, int32_t n, const int32_t* converged,
                                         double rho, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!mt_state || !converged || !out))) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  synthetic_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(mt_state, n, converged, rho, out);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_confused_level(uint32_t* mt_state, int32_t n, const int32_t* true_level,
                                      const double* matrix, int32_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!mt_state || !true_level || !matrix || !out))) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  confusion_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(mt_state, n, true_level, matrix, out);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_early_termination(const double* history, const int32_t* offsets,
                                         int32_t n_sets, double threshold, int32_t rounds,
                                         int32_t* out, void* stream) {
  if (n_sets < 0 || rounds < 1 || (n_sets > 0 && (!history || !offsets || !out))) return DUCHESS_EINVAL;
  if (n_sets == 0) return DUCHESS_OK;
  streak_kernel<<<(n_sets + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      history, offsets, n_sets, threshold, rounds, out);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_confused_levels(const uint32_t* mt_states, int32_t n,
                                       const int32_t* true_level, const double* matrix,
                                       int32_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!mt_states || !true_level || !matrix || !out))) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  confusion_streams_kernel<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      mt_states, n, true_level, matrix, out);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_timeline(const int32_t* round_rec, int32_t n_slots, double ms_per_token,
                                double ms_per_extra_branch, int64_t probe_cost_ms,
                                int64_t* service_ms, int64_t* first_token_ms, void* stream) {
  if (n_slots < 0 || (n_slots > 0 && (!round_rec || !service_ms || !first_token_ms)))
    return DUCHESS_EINVAL;
  if (n_slots == 0) return DUCHESS_OK;
  timeline_kernel<<<(n_slots + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      round_rec, n_slots, ms_per_token, ms_per_extra_branch, (long long)probe_cost_ms,
      reinterpret_cast<long long*>(service_ms), reinterpret_cast<long long*>(first_token_ms));
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_mt_seed(const uint64_t* seeds, int32_t n, uint32_t* out_states, void* stream) {
  if (n < 0 || (n > 0 && (!seeds || !out_states))) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  mt_seed_kernel<<<(n + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(seeds, n, out_states);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
