// K1 core shared by the stand-alone scorer (score.cu) and the fused round
// kernel (decide.cu, duchess_step): the TMA-bulk producer loop and the
// consumer-warp pooling + LayerNorm + probe dot of one window.
//
// Restates the reference's linear-probe forward `mlp_forward`
// (pkg/src/branchsim/predictor.py:126-151) over a token-pooled window:
//     m     = mean_t x[t, :]                       (pooling: north-star extension)
//     z     = (m - mean(m)) / sqrt(var(m) + 1e-5)  (predictor.py:134-136, population var)
//     logit = sum_h w_h (g_h z_h + b_h) + b        (predictor.py:137-138, :146)
//     prob  = clip(sigmoid(logit), 1e-12, 1-1e-12) (predictor.py:148)
// folded as logit = (sum_h wg_h (m_h - mu)) / sigma + c1.
//
// All fp32 arithmetic below uses explicit _rn intrinsics, so the two
// translation units (score.cu default, decide.cu --fmad=false) produce the
// same bits for the same window.
#pragma once
#include "common.cuh"

namespace duchess {

struct ScoreArgs {
  const char* acts;
  int64_t row_stride, layer_stride, token_stride;  // elements
  int64_t n_units;                                 // rows * L
  int L, T, H;
  int nsplit, chunk;                               // chunk = columns per split
  const float* wg;
  const float* c1;
  const uint8_t* mask;
  float* out_logit;
  double* out_prob;
  float4* partials;     // [n_units * nsplit] (mean, M2, dot, wsum)
  unsigned* counters;   // [n_units]
};

__device__ __forceinline__ void write_score(const ScoreArgs& a, int64_t unit, float logit) {
  a.out_logit[unit] = logit;
  double p = 1.0 / (1.0 + exp(-double(logit)));
  p = fmin(fmax(p, kProbClip), 1.0 - kProbClip);
  a.out_prob[unit] = p;
}

// ---------------------------------------------------------------------------
// Persistent warp-specialised scorer: a producer warp streams each window's
// token rows into a shared-memory ring with cp.async.bulk (mbarrier
// transaction counts, L2 evict-first), 8 consumer warps pool from shared
// memory and finish the window (two-pass LN stats + dot) while the producer
// already streams the next one. Units are assigned round-robin over the grid
// (unit u -> CTA u % gridDim.x) in list order.
constexpr int kTmaConsWarps = 8;
constexpr int kTmaCons = kTmaConsWarps * 32;
constexpr int kTmaStageTarget = 8 * 1024;     // fused step kernel; row-size bound (4x) of the TMA path
constexpr int kScoreStageTarget = 32 * 1024;  // stand-alone scorer's stage (bulk copy) target
constexpr int kTmaSmemBudget = 196 * 1024;

struct TmaArgs {
  const int32_t* row_list;   // nullable
  const int32_t* row_count;  // device count when row_list != nullptr
  const int32_t* row_par;    // nullable: double-buffered list, parity word
  int64_t list_stride;       // entries per parity buffer (with row_par)
  int tokens_per_stage;
  int stages;
  int row_bytes;             // H * esz
  int contiguous;            // token_stride == H
  int no_input_wait;         // DUCHESS_SCORE_NO_INPUT_WAIT: see k1_begin
};

// Programmatic dependent launch protocol of the scorers. By default the
// inputs (survivor list, windows) are read after griddepcontrol.wait, i.e.
// after the preceding kernel in the stream completed. With no_input_wait the
// inputs were final before that kernel even started (it is another request
// shard's round), so streaming starts at once and the wait moves to the end:
// this grid still completes only after its predecessor.
__device__ __forceinline__ void k1_begin(const TmaArgs& t) {
  if (!t.no_input_wait) pdl_wait();
  pdl_launch_dependents();
}
__device__ __forceinline__ void k1_end(const TmaArgs& t) {
  if (t.no_input_wait && threadIdx.x == 0) pdl_wait();
}

struct TmaRing {
  char* ring;
  uint64_t* full_bar;
  uint64_t* empty_bar;
  int stage_bytes;
};

__device__ __forceinline__ bool tma_unit(const ScoreArgs& a, const TmaArgs& t, int64_t u,
                                         int64_t& row, int& l) {
  const int64_t r = u / a.L;
  l = int(u - r * a.L);
  if (t.row_list) {
    row = t.row_list[r];
    return true;
  }
  row = r;
  return a.mask == nullptr || a.mask[r] != 0;
}

__device__ __forceinline__ void tma_ring_init(const TmaArgs& t, TmaRing& rg) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < t.stages; ++s) {
      mbar_init(&rg.full_bar[s], 1);
      mbar_init(&rg.empty_bar[s], kTmaConsWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// Producer (one elected lane): stream every unit of this CTA into the ring.
template <int ESZ>
__device__ __forceinline__ void tma_produce(const ScoreArgs& a, const TmaArgs& t, const TmaRing& rg,
                                            int64_t n_units) {
  const uint64_t pol = evict_first_policy();
  int s = 0;
  uint32_t ph = 0;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    int64_t row;
    int l;
    if (!tma_unit(a, t, u, row, l)) continue;
    const char* base = a.acts + (row * a.row_stride + int64_t(l) * a.layer_stride) * ESZ;
    for (int t0 = 0; t0 < a.T; t0 += t.tokens_per_stage) {
      const int nt = min(t.tokens_per_stage, a.T - t0);
      mbar_wait(&rg.empty_bar[s], ph ^ 1u);
      mbar_expect_tx(&rg.full_bar[s], uint32_t(nt * t.row_bytes));
      char* dst = rg.ring + size_t(s) * rg.stage_bytes;
      if (t.contiguous) {
        bulk_g2s(dst, base + int64_t(t0) * t.row_bytes, uint32_t(nt * t.row_bytes),
                 &rg.full_bar[s], pol);
      } else {
        for (int k = 0; k < nt; ++k)
          bulk_g2s(dst + k * t.row_bytes, base + int64_t(t0 + k) * a.token_stride * ESZ,
                   uint32_t(t.row_bytes), &rg.full_bar[s], pol);
      }
      if (++s == t.stages) { s = 0; ph ^= 1u; }
    }
  }
}

// Block reduction over the 8 consumer warps (named barrier 1); red is double
// buffered so one barrier per reduction suffices.
__device__ __forceinline__ void cons_sum2(float& x, float& y, float2 (*red)[kTmaConsWarps], int& k) {
  x = warp_sum(x);
  y = warp_sum(y);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[k & 1][warp] = make_float2(x, y);
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaCons) : "memory");
  float sx = 0.f, sy = 0.f;
#pragma unroll
  for (int w = 0; w < kTmaConsWarps; ++w) {
    sx = __fadd_rn(sx, red[k & 1][w].x);
    sy = __fadd_rn(sy, red[k & 1][w].y);
  }
  x = sx;
  y = sy;
  ++k;
}

// Consumers (threads 0..kTmaCons-1): score every unit of this CTA; after a
// unit's score is written, thread 0 calls done(row, l, unit).
template <bool BF16, int VPT, typename Done>
__device__ __forceinline__ void tma_consume(const ScoreArgs& a, const TmaArgs& t, const TmaRing& rg,
                                            int64_t n_units, float2 (*red)[kTmaConsWarps],
                                            Done done) {
  constexpr int VEC = BF16 ? 8 : 4;
  const int lane = threadIdx.x & 31;
  const int nvec = t.row_bytes / 16;
  int s = 0, k = 0;
  uint32_t ph = 0;
  const float invT = 1.0f / float(a.T);
  const bool pow2T = (a.T & (a.T - 1)) == 0;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    int64_t row;
    int l;
    if (!tma_unit(a, t, u, row, l)) continue;
    float acc[VPT][VEC];
#pragma unroll
    for (int j = 0; j < VPT; ++j)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[j][v] = 0.f;
    for (int t0 = 0; t0 < a.T; t0 += t.tokens_per_stage) {
      const int nt = min(t.tokens_per_stage, a.T - t0);
      mbar_wait(&rg.full_bar[s], ph);
      const char* st = rg.ring + size_t(s) * rg.stage_bytes;
      for (int q = 0; q < nt; ++q) {
        const uint4* rowv = reinterpret_cast<const uint4*>(st + q * t.row_bytes);
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          const int v = j * kTmaCons + int(threadIdx.x);
          if (v < nvec) {
            const uint4 x = rowv[v];
            const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
            if constexpr (BF16) {
#pragma unroll
              for (int e = 0; e < 4; ++e) add_bf16x2_f32(acc[j][2 * e], acc[j][2 * e + 1], w4[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[j][e] = __fadd_rn(acc[j][e], __uint_as_float(w4[e]));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rg.empty_bar[s]);
      if (++s == t.stages) { s = 0; ph ^= 1u; }
    }
    const float* wrow = a.wg + int64_t(l) * a.H;
    float s1 = 0.f, unused = 0.f;
    // window mean: exact scaling for a power-of-two T (none for T = 1), IEEE
    // division otherwise; a uniform branch, so the division is not evaluated
    // (and discarded by a select) when T is a power of two
    if (!pow2T) {
#pragma unroll
      for (int j = 0; j < VPT; ++j)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[j][e] = __fdiv_rn(acc[j][e], float(a.T));
    } else if (a.T != 1) {
#pragma unroll
      for (int j = 0; j < VPT; ++j)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[j][e] = __fmul_rn(acc[j][e], invT);
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int v = j * kTmaCons + int(threadIdx.x);
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (v < nvec) s1 = __fadd_rn(s1, acc[j][e]);
    }
    cons_sum2(s1, unused, red, k);
    const float mean = __fdiv_rn(s1, float(a.H));
    // second pass: centred square sum and probe dot, one packed FFMA2 per
    // element ({c*c + qq, w*c + d}); the folded weights come from L1/L2
    float qq = 0.f, d = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int v = j * kTmaCons + int(threadIdx.x);
      if (v < nvec) {
        const float4* w4 = reinterpret_cast<const float4*>(wrow + v * VEC);
        float wv[VEC];
#pragma unroll
        for (int q = 0; q < VEC / 4; ++q) {
          const float4 t4 = __ldg(w4 + q);
          wv[4 * q] = t4.x; wv[4 * q + 1] = t4.y; wv[4 * q + 2] = t4.z; wv[4 * q + 3] = t4.w;
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const float c = __fsub_rn(acc[j][e], mean);
          ffma2(qq, d, c, wv[e], c, c);
        }
      }
    }
    cons_sum2(qq, d, red, k);
    if (threadIdx.x == 0) {
      const float var = __fdiv_rn(qq, float(a.H));
      const float logit = __fadd_rn(__fdiv_rn(d, __fsqrt_rn(__fadd_rn(var, kLayerNormEps))), a.c1[l]);
      const int64_t unit = row * a.L + l;
      write_score(a, unit, logit);
      done(row, l, unit);
    }
  }
}

}  // namespace duchess
