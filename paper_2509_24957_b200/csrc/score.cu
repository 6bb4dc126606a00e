// K1: fused token-pooling + LayerNorm + linear-probe scoring (sm_100a).
//
// Restates, batched over every active (branch, layer) window, the reference's
// per-vector probe forward `mlp_forward` (reference pkg/src/branchsim/
// predictor.py:126-151) for the linear probe (layer_dims = [], head_dim = 1):
//     m      = mean_t x[t, :]                        (pooling: north-star extension)
//     z      = (m - mean(m)) / sqrt(var(m) + 1e-5)   (predictor.py:134-136, population var)
//     logit  = sum_h w_h (g_h z_h + b_h) + b          (predictor.py:137-138, :146)
//     prob   = clip(sigmoid(logit), 1e-12, 1-1e-12)   (predictor.py:148)
// folded as logit = (sum_h wg_h (m_h - mu)) / sigma + c1 with wg = w*g and
// c1 = sum w*b_ln + b precomputed on the host.
//
// The kernel is HBM-bound (< 1 FLOP/B): each CTA streams one H-chunk of one
// window with 128-bit no-L1-allocate loads, keeps its pooled values in
// registers (two-pass mean/variance costs no extra HBM traffic) and, when a
// window is split over several CTAs, merges (count, mean, M2, dot) partials
// with Chan's formula in fixed chunk order in the last-arriving CTA, so the
// result is deterministic run to run.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "score_core.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

template <int NT>
__device__ __forceinline__ void block_sum2(float& a, float& b, float2* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = make_float2(a, b);
  __syncthreads();
  if (warp == 0) {
    float2 v = lane < NT / 32 ? red[lane] : make_float2(0.f, 0.f);
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    if (lane == 0) red[NT / 32] = v;
  }
  __syncthreads();
  a = red[NT / 32].x;
  b = red[NT / 32].y;
  __syncthreads();
}

// Last CTA of a split window: merge chunk partials in chunk order (double).
__device__ void merge_partials(const ScoreArgs& a, int64_t unit, int l) {
  const float4* parts = a.partials + unit * a.nsplit;
  double n_a = 0.0, mean = 0.0, m2 = 0.0;
  for (int k = 0; k < a.nsplit; ++k) {
    float4 pk = __ldcg(parts + k);
    int beg = k * a.chunk, end = min(a.H, beg + a.chunk);
    double n_b = double(end - beg);
    if (n_b <= 0) continue;
    double delta = double(pk.x) - mean;
    double n = n_a + n_b;
    mean += delta * n_b / n;
    m2 += double(pk.y) + delta * delta * n_a * n_b / n;
    n_a = n;
  }
  double dot = 0.0;
  for (int k = 0; k < a.nsplit; ++k) {
    float4 pk = __ldcg(parts + k);
    int beg = k * a.chunk, end = min(a.H, beg + a.chunk);
    if (end <= beg) continue;
    dot += double(pk.z) + (double(pk.x) - mean) * double(pk.w);
  }
  double var = m2 / double(a.H);
  float logit = float(dot / sqrt(var + double(kLayerNormEps))) + a.c1[l];
  write_score(a, unit, logit);
}

// Fast path: 16-byte aligned windows, H a multiple of the vector width.
template <bool BF16, int NT, int PASSES>
__global__ void __launch_bounds__(NT) score_fast_kernel(ScoreArgs a) {
  constexpr int VEC = BF16 ? 8 : 4;                 // elements per 16-byte load
  constexpr int ESZ = BF16 ? 2 : 4;
  constexpr int U = (16 / PASSES) > 0 ? (16 / PASSES) : 1;  // tokens per load batch
  __shared__ float2 red[NT / 32 + 1];
  __shared__ int last_flag;

  const int64_t unit = blockIdx.x / a.nsplit;
  const int split = blockIdx.x - int(unit * a.nsplit);
  const int64_t row = unit / a.L;
  const int l = int(unit - row * a.L);
  if (a.mask != nullptr && a.mask[row] == 0) return;

  const int cbeg = split * a.chunk;
  const int cend = min(a.H, cbeg + a.chunk);
  const char* base = a.acts + (row * a.row_stride + int64_t(l) * a.layer_stride) * ESZ;
  const int64_t tok_bytes = a.token_stride * ESZ;

  float acc[PASSES][VEC];
  bool valid[PASSES];
  const char* colp[PASSES];
#pragma unroll
  for (int p = 0; p < PASSES; ++p) {
    const int col = cbeg + (p * NT + int(threadIdx.x)) * VEC;
    valid[p] = col < cend;
    colp[p] = base + int64_t(col) * ESZ;
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[p][v] = 0.f;
  }

  for (int t0 = 0; t0 < a.T; t0 += U) {
    uint4 buf[U][PASSES];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int p = 0; p < PASSES; ++p)
        if (valid[p] && t0 + u < a.T) buf[u][p] = ldg_stream(colp[p] + int64_t(t0 + u) * tok_bytes);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int p = 0; p < PASSES; ++p)
        if (valid[p] && t0 + u < a.T) {
          const uint32_t w[4] = {buf[u][p].x, buf[u][p].y, buf[u][p].z, buf[u][p].w};
          if constexpr (BF16) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[p][2 * q] += bf16lo(w[q]);
              acc[p][2 * q + 1] += bf16hi(w[q]);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] += __uint_as_float(w[q]);
          }
        }
  }

  // Pooled window mean, local (chunk) statistics.
  const float invT = 1.0f / float(a.T);
  float wgv[PASSES][VEC];
  float s1 = 0.f, sw = 0.f;
  const float* wrow = a.wg + int64_t(l) * a.H;
  if ((a.T & (a.T - 1)) != 0) {     // uniform branch: no discarded division
#pragma unroll
    for (int p = 0; p < PASSES; ++p)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[p][v] = acc[p][v] / float(a.T);
  } else if (a.T != 1) {
#pragma unroll
    for (int p = 0; p < PASSES; ++p)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[p][v] = acc[p][v] * invT;
  }
#pragma unroll
  for (int p = 0; p < PASSES; ++p) {
    const int col = cbeg + (p * NT + int(threadIdx.x)) * VEC;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      wgv[p][v] = valid[p] ? __ldg(wrow + col + v) : 0.f;
      if (valid[p]) { s1 += acc[p][v]; sw += wgv[p][v]; }
    }
  }
  block_sum2<NT>(s1, sw, red);
  const float n_loc = float(cend - cbeg);
  const float mean_loc = s1 / n_loc;
  float q = 0.f, d = 0.f;
#pragma unroll
  for (int p = 0; p < PASSES; ++p)
#pragma unroll
    for (int v = 0; v < VEC; ++v)
      if (valid[p]) {
        const float c = acc[p][v] - mean_loc;
        q += c * c;
        d += wgv[p][v] * c;
      }
  block_sum2<NT>(q, d, red);

  if (a.nsplit == 1) {
    if (threadIdx.x == 0) {
      const float var = q / float(a.H);
      write_score(a, unit, d / sqrtf(var + kLayerNormEps) + a.c1[l]);
    }
    return;
  }
  if (threadIdx.x == 0) {
    a.partials[unit * a.nsplit + split] = make_float4(mean_loc, q, d, sw);
    __threadfence();
    const unsigned prev = atomicAdd(a.counters + unit, 1u);
    last_flag = (prev == unsigned(a.nsplit - 1));
  }
  __syncthreads();
  if (last_flag && threadIdx.x == 0) {
    __threadfence();
    merge_partials(a, unit, l);
    a.counters[unit] = 0u;   // ready for the next launch
  }
}

// Generic path: any alignment / width; pooled window staged in shared memory.
template <bool BF16>
__global__ void __launch_bounds__(256) score_generic_kernel(ScoreArgs a) {
  constexpr int NT = 256;
  extern __shared__ float pooled[];
  __shared__ float2 red[NT / 32 + 1];
  const int64_t unit = blockIdx.x;
  const int64_t row = unit / a.L;
  const int l = int(unit - row * a.L);
  if (a.mask != nullptr && a.mask[row] == 0) return;
  const int64_t off = row * a.row_stride + int64_t(l) * a.layer_stride;
  const float* wrow = a.wg + int64_t(l) * a.H;
  float s1 = 0.f, sw = 0.f;
  for (int h = threadIdx.x; h < a.H; h += NT) {
    float acc = 0.f;
    for (int t = 0; t < a.T; ++t) {
      const int64_t idx = off + int64_t(t) * a.token_stride + h;
      if constexpr (BF16) {
        const uint16_t raw = reinterpret_cast<const uint16_t*>(a.acts)[idx];
        acc += __uint_as_float(uint32_t(raw) << 16);
      } else {
        acc += reinterpret_cast<const float*>(a.acts)[idx];
      }
    }
    const float m = acc / float(a.T);
    pooled[h] = m;
    s1 += m;
    sw += wrow[h];
  }
  block_sum2<NT>(s1, sw, red);
  const float mean = s1 / float(a.H);
  float q = 0.f, d = 0.f;
  for (int h = threadIdx.x; h < a.H; h += NT) {
    const float c = pooled[h] - mean;
    q += c * c;
    d += wrow[h] * c;
  }
  block_sum2<NT>(q, d, red);
  if (threadIdx.x == 0) {
    const float var = q / float(a.H);
    write_score(a, unit, d / sqrtf(var + kLayerNormEps) + a.c1[l]);
  }
}

// ---------------------------------------------------------------------------
// Persistent warp-specialised variant (score_core.cuh): one producer warp
// streams windows into a shared-memory ring with cp.async.bulk, 8 consumer
// warps pool + LayerNorm + dot. Windows come from a compacted row list
// (written by duchess_advance) or from all rows filtered by the mask.
template <bool BF16, int VPT>
__global__ void __launch_bounds__(kTmaCons + 32, 2) score_tma_kernel(ScoreArgs a, TmaArgs t) {
  constexpr int ESZ = BF16 ? 2 : 4;
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full_bar[32], empty_bar[32];
  __shared__ float2 red[2][kTmaConsWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TmaRing rg{ring, full_bar, empty_bar, t.tokens_per_stage * t.row_bytes};
  tma_ring_init(t, rg);
  __syncthreads();
  // setup above overlaps the previous kernel; inputs are read below. Then let
  // the next launch (duchess_round) become resident and prefetch its state
  // while this one streams.
  k1_begin(t);
  if (t.row_par) {                     // engine list: the parity duchess_round left
    const int par = *t.row_par;
    t.row_list += par * t.list_stride;
    t.row_count += par;
  }
  const int64_t n_units = (t.row_list ? int64_t(*t.row_count) : a.n_units / a.L) * a.L;
  if (warp == kTmaConsWarps) {
    if (lane == 0) tma_produce<ESZ>(a, t, rg, n_units);
    return;
  }
  tma_consume<BF16, VPT>(a, t, rg, n_units, red, [](int64_t, int, int64_t) {});
  k1_end(t);                           // thread 0 is a consumer
}

template <bool BF16>
static cudaError_t launch_tma(const ScoreArgs& a, const TmaArgs& t, int vpt, int grid, cudaStream_t s) {
  const size_t smem = size_t(t.stages) * t.tokens_per_stage * t.row_bytes;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTmaCons + 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a, t);
  };
  switch (vpt) {
    case 1: go(score_tma_kernel<BF16, 1>); break;
    case 2: go(score_tma_kernel<BF16, 2>); break;
    case 4: go(score_tma_kernel<BF16, 4>); break;
    case 8: go(score_tma_kernel<BF16, 8>); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}


// Last-token windows (T = 1: the paper's probe reads one token, PAPER.md:150;
// C1 and C3-T1). A unit is one H-vector (10 KB at H = 5120 bf16), too small
// for a CTA-wide LayerNorm reduction: each WARP scores whole units. A lane
// issues all of its NV 16-byte loads of the unit at once (L1 no-allocate), so
// 16 warps x 10 KB per SM are in flight; the two-pass LN statistics run on the
// registers (exact centring, no second read) and the folded probe weights of
// all layers sit in shared memory. Units are dealt round-robin over the grid's
// warps; no CTA barrier after the weight load.
constexpr int kRowsWarps = 16;
constexpr int kRowsSmemMax = 160 * 1024;
template <bool BF16, int NV, bool WSMEM>
__global__ void __launch_bounds__(kRowsWarps * 32, 1) score_rows_kernel(ScoreArgs a, TmaArgs t) {
  constexpr int VEC = BF16 ? 8 : 4;
  constexpr int ESZ = BF16 ? 2 : 4;
  extern __shared__ __align__(16) float wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = t.row_bytes / 16;
  if constexpr (WSMEM) {      // the folded weights are not written by the previous kernel
    const int nw = a.L * a.H / 4;
    for (int i = threadIdx.x; i < nw; i += blockDim.x)
      reinterpret_cast<float4*>(wsm)[i] = __ldg(reinterpret_cast<const float4*>(a.wg) + i);
    __syncthreads();
  }
  k1_begin(t);
  if (t.row_par) {
    const int par = *t.row_par;
    t.row_list += par * t.list_stride;
    t.row_count += par;
  }
  const int64_t n_units = (t.row_list ? int64_t(*t.row_count) : a.n_units / a.L) * a.L;
  const int64_t gw = int64_t(blockIdx.x) * kRowsWarps + warp;
  const int64_t nw = int64_t(gridDim.x) * kRowsWarps;
  auto unit_src = [&](int64_t row, int l) {
    return reinterpret_cast<const uint4*>(a.acts + (row * a.row_stride + int64_t(l) * a.layer_stride) * ESZ);
  };
  // next valid unit of this warp at or after u (n_units if none)
  auto next_unit = [&](int64_t u, int64_t& row, int& l) {
    for (; u < n_units; u += nw)
      if (tma_unit(a, t, u, row, l)) return u;
    return n_units;
  };
  auto load = [&](uint4 (&xv)[NV], int j, const uint4* src) {
    const int v = j * 32 + lane;
    xv[j] = v < nvec ? ldg_stream(src + v) : make_uint4(0u, 0u, 0u, 0u);
  };
  int64_t row = 0;
  int l = 0;
  int64_t u = next_unit(gw, row, l);
  uint4 xv[NV];
  if (u < n_units) {
#pragma unroll
    for (int j = 0; j < NV; ++j) load(xv, j, unit_src(row, l));
  }
  // Rolling register pipeline: pass 2 of unit k reloads each vector register
  // with unit k+1's data right after its last use, so the next unit's loads
  // are in flight during pass 2 and the reductions.
  while (u < n_units) {
    // pass 1: eight independent chains; bf16 pairs are added straight into fp32
    // (FHADD), so no converted copy of the vector stays live into pass 2
    float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint32_t w4[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
      if constexpr (BF16) {
#pragma unroll
        for (int e = 0; e < 4; ++e) add_bf16x2_f32(s8[2 * e], s8[2 * e + 1], w4[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) s8[e] = __fadd_rn(s8[e], __uint_as_float(w4[e]));
      }
    }
#pragma unroll
    for (int e = 1; e < 8; e <<= 1)
#pragma unroll
      for (int q = 0; q < 8; q += 2 * e) s8[q] = __fadd_rn(s8[q], s8[q + e]);
    const float s1 = warp_sum(s8[0]);
    const float mean = __fdiv_rn(s1, float(a.H));
    int64_t nrow = 0;
    int nl = 0;
    const int64_t un = next_unit(u + nw, nrow, nl);
    const uint4* nsrc = un < n_units ? unit_src(nrow, nl) : nullptr;
    const float* wrow = (WSMEM ? wsm : a.wg) + int64_t(l) * a.H;
    float qq = 0.f, d = 0.f, qq2 = 0.f, d2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int v = j * 32 + lane;
      if (v < nvec) {
        const uint32_t w4[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
        // centred values c = x - mean, rounded once: for bf16 one mixed-precision
        // add per element straight from the packed pair (FHADD, no conversion)
        float c[VEC];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (BF16) {
            c[2 * e] = -mean;
            c[2 * e + 1] = -mean;
            add_bf16x2_f32(c[2 * e], c[2 * e + 1], w4[e]);
          } else {
            c[e] = __fsub_rn(__uint_as_float(w4[e]), mean);
          }
        }
        if (nsrc) load(xv, j, nsrc);
        const float4* wp = reinterpret_cast<const float4*>(wrow + v * VEC);
#pragma unroll
        for (int q = 0; q < VEC / 4; ++q) {
          const float4 t4 = WSMEM ? wp[q] : __ldg(wp + q);
          ffma2(qq, d, c[4 * q], t4.x, c[4 * q], c[4 * q]);
          ffma2(qq2, d2, c[4 * q + 1], t4.y, c[4 * q + 1], c[4 * q + 1]);
          ffma2(qq, d, c[4 * q + 2], t4.z, c[4 * q + 2], c[4 * q + 2]);
          ffma2(qq2, d2, c[4 * q + 3], t4.w, c[4 * q + 3], c[4 * q + 3]);
        }
      } else if (nsrc) {
        load(xv, j, nsrc);
      }
    }
    qq = warp_sum(__fadd_rn(qq, qq2));
    d = warp_sum(__fadd_rn(d, d2));
    if (lane == 0) {
      const float var = __fdiv_rn(qq, float(a.H));
      const float logit = __fadd_rn(__fdiv_rn(d, __fsqrt_rn(__fadd_rn(var, kLayerNormEps))), a.c1[l]);
      write_score(a, row * a.L + l, logit);
    }
    u = un;
    row = nrow;
    l = nl;
  }
  k1_end(t);
}

// Last-token windows, bulk-copy variant (default). Same per-window arithmetic
// as score_rows_kernel (warp per window, two-pass LN statistics on registers),
// restructured around the memory pipe:
//  * each warp owns one shared-memory slot that a single cp.async.bulk fills
//    with its NEXT window: right after the warp has copied window k from the
//    slot into registers, lane 0 refills the slot with window k+1, so one
//    window per warp is in flight for the whole time the warp pools, reduces
//    and scores window k;
//  * a CTA scores one probe layer (CTA b: layer b % L), so only that layer's
//    folded weights (H floats) sit in shared memory and the rest of the 227 KB
//    holds slots: 16 warps x one 10 KB window in flight per SM at H = 5120;
//  * a warp's windows are taken in batches of 32: lane i holds the row of the
//    batch's window i (one list load per lane per batch, fetched a batch ahead)
//    and, once scored, its LN sums, so list loads and the fp64 sigmoid run once
//    per 32 windows spread over the lanes, not on the per-window chain;
//  * pass 2 runs on element pairs: two FHADD produce c = x - mean into an
//    aligned register pair, then {qq} += c*c and {d} += w*c are packed FFMA2.
constexpr int kBulkSlotAlign = 128;
template <bool BF16, int NV, bool FULL>
__global__ void __launch_bounds__(kRowsWarps * 32, 1) score_rows_bulk_kernel(ScoreArgs a, TmaArgs t,
                                                                          int wbytes, int slot_bytes) {
  constexpr int VEC = BF16 ? 8 : 4;
  constexpr int ESZ = BF16 ? 2 : 4;
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[kRowsWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int nvec = t.row_bytes / 16;
  const int l = int(blockIdx.x % unsigned(a.L));                 // this CTA's probe layer
  const int64_t grp = blockIdx.x / unsigned(a.L), ngrp = gridDim.x / unsigned(a.L);
  float* wsm = reinterpret_cast<float*>(smem);
  char* slot = smem + wbytes + warp * slot_bytes;
  {
    // the layer's weights as VEC/4 planes (float4 q of vector v at plane q,
    // index v), so a warp's 128-bit weight reads are contiguous (conflict-free)
    const int per_layer = a.H / 4;
    const float4* src = reinterpret_cast<const float4*>(a.wg) + int64_t(l) * per_layer;
    for (int k = threadIdx.x; k < per_layer; k += blockDim.x) {
      const int v = k / (VEC / 4), q = k - v * (VEC / 4);
      reinterpret_cast<float4*>(wsm)[q * nvec + v] = __ldg(src + k);
    }
    if (lane == 0) {
      mbar_init(&bar[warp], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  k1_begin(t);
  if (t.row_par) {
    const int par = *t.row_par;
    t.row_list += par * t.list_stride;
    t.row_count += par;
  }
  const int64_t n_rows = t.row_list ? int64_t(*t.row_count) : a.n_units / a.L;
  const int64_t nw = ngrp * nwarps;                 // warps scoring this layer
  const int64_t bstride = 32 * nw;
  const uint64_t pol = evict_first_policy();
  // entry r of the warp's sequence r = gw + k * nw (list entry or masked row)
  auto load_batch = [&](int64_t base, int64_t& row) -> unsigned {
    const int64_t r = base + int64_t(lane) * nw;
    row = 0;
    bool ok = r < n_rows;
    if (ok) {
      if (t.row_list) {
        row = t.row_list[r];
      } else {
        row = r;
        ok = a.mask == nullptr || a.mask[r] != 0;
      }
    }
    return __ballot_sync(0xffffffffu, ok);
  };
  auto refill = [&](int64_t row) {
    mbar_expect_tx(&bar[warp], uint32_t(t.row_bytes));
    bulk_g2s(slot, a.acts + (row * a.row_stride + int64_t(l) * a.layer_stride) * ESZ,
             uint32_t(t.row_bytes), &bar[warp], pol);
  };
  int64_t base = grp * nwarps + warp;
  int64_t rowc, rown;
  unsigned mc = load_batch(base, rowc);
  unsigned mn = load_batch(base + bstride, rown);
  auto shift = [&]() {
    base += bstride;
    rowc = rown;
    mc = mn;
    mn = load_batch(base + bstride, rown);
  };
  while (mc == 0 && base < n_rows) shift();         // (mask path) skip empty batches
  int i = mc ? __ffs(mc) - 1 : 0;
  if (mc) {
    const int64_t r0 = __shfl_sync(0xffffffffu, rowc, i);
    if (lane == 0) refill(r0);
  }
  float my_q = 0.f, my_d = 0.f;
  uint32_t ph = 0;
  const uint4* s4 = reinterpret_cast<const uint4*>(slot);
  const float c1 = a.c1[l];
  while (mc) {
    const unsigned rest = mc & ~((2u << i) - 1u);     // later windows of this batch
    bool have_next = true;
    int64_t nrow = 0;
    if (rest) nrow = __shfl_sync(0xffffffffu, rowc, __ffs(rest) - 1);
    else if (mn) nrow = __shfl_sync(0xffffffffu, rown, __ffs(mn) - 1);
    else have_next = false;
    mbar_wait(&bar[warp], ph);
    ph ^= 1u;
    uint4 xv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int v = j * 32 + lane;
      xv[j] = (FULL || v < nvec) ? s4[v] : make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();
    if (lane == 0 && have_next) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // slot reads before the refill
      refill(nrow);
    }
    // pass 1: eight independent chains (FHADD straight from the packed pair)
    float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint32_t w4[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
      if constexpr (BF16) {
#pragma unroll
        for (int e = 0; e < 4; ++e) add_bf16x2_f32(s8[2 * e], s8[2 * e + 1], w4[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) s8[e] = __fadd_rn(s8[e], __uint_as_float(w4[e]));
      }
    }
#pragma unroll
    for (int e = 1; e < 8; e <<= 1)
#pragma unroll
      for (int q = 0; q < 8; q += 2 * e) s8[q] = __fadd_rn(s8[q], s8[q + e]);
    const float s1 = warp_sum(s8[0]);
    const float mean = __fdiv_rn(s1, float(a.H));
    // pass 2 on element pairs
    unsigned long long qa = 0ull, qb = 0ull, da = 0ull, db = 0ull;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int v = j * 32 + lane;
      if (FULL || v < nvec) {
        const uint32_t w4[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
        const float4* wp = reinterpret_cast<const float4*>(wsm) + v;
#pragma unroll
        for (int q = 0; q < VEC / 4; ++q) {
          const float4 t4 = wp[q * nvec];
          float c0, c1_, c2, c3;
          if constexpr (BF16) {
            c0 = -mean; c1_ = -mean; c2 = -mean; c3 = -mean;
            add_bf16x2_f32(c0, c1_, w4[2 * q]);
            add_bf16x2_f32(c2, c3, w4[2 * q + 1]);
          } else {
            c0 = __fsub_rn(__uint_as_float(w4[0]), mean);
            c1_ = __fsub_rn(__uint_as_float(w4[1]), mean);
            c2 = __fsub_rn(__uint_as_float(w4[2]), mean);
            c3 = __fsub_rn(__uint_as_float(w4[3]), mean);
          }
          const unsigned long long cA = pack_f32x2(c0, c1_), cB = pack_f32x2(c2, c3);
          fma_f32x2(qa, cA, cA);
          fma_f32x2(qb, cB, cB);
          fma_f32x2(da, cA, pack_f32x2(t4.x, t4.y));
          fma_f32x2(db, cB, pack_f32x2(t4.z, t4.w));
        }
      }
    }
    float q0, q1, q2, q3, d0, d1, d2, d3;
    unpack_f32x2(qa, q0, q1);
    unpack_f32x2(qb, q2, q3);
    unpack_f32x2(da, d0, d1);
    unpack_f32x2(db, d2, d3);
    const float qq = warp_sum(__fadd_rn(__fadd_rn(q0, q1), __fadd_rn(q2, q3)));
    const float d = warp_sum(__fadd_rn(__fadd_rn(d0, d1), __fadd_rn(d2, d3)));
    if (lane == i) {               // the butterfly leaves the sums in every lane
      my_q = qq;
      my_d = d;
    }
    if (rest) {
      i = __ffs(rest) - 1;
      continue;
    }
    // batch complete: every lane finishes its own window (LN scale, logit, sigmoid)
    if ((mc >> lane) & 1u) {
      const float var = __fdiv_rn(my_q, float(a.H));
      const float logit = __fadd_rn(__fdiv_rn(my_d, __fsqrt_rn(__fadd_rn(var, kLayerNormEps))), c1);
      write_score(a, rowc * a.L + l, logit);
    }
    shift();
    if (!have_next) {
      while (mc == 0 && base < n_rows) shift();
      if (mc) {
        i = __ffs(mc) - 1;
        const int64_t r0 = __shfl_sync(0xffffffffu, rowc, i);
        if (lane == 0) refill(r0);
      }
    } else {
      i = __ffs(mc) - 1;
    }
  }
  k1_end(t);
}

// Shared-memory plan of score_rows_bulk_kernel: warps that fit beside the weights.
static int rows_bulk_warps(int64_t wbytes, int64_t row_bytes, int smem_max, int& slot_bytes) {
  slot_bytes = int((row_bytes + kBulkSlotAlign - 1) / kBulkSlotAlign * kBulkSlotAlign);
  const int64_t room = int64_t(smem_max) - wbytes;
  if (room < slot_bytes) return 0;
  return int(room / slot_bytes < kRowsWarps ? room / slot_bytes : kRowsWarps);
}

template <bool BF16>
static cudaError_t launch_rows_bulk(const ScoreArgs& a, const TmaArgs& t, int nv, int grid,
                                    int nwarps, int slot_bytes, cudaStream_t s) {
  const int wbytes = (a.H * int(sizeof(float)) + kBulkSlotAlign - 1) / kBulkSlotAlign * kBulkSlotAlign;
  const size_t smem = size_t(wbytes) + size_t(nwarps) * slot_bytes;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nwarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a, t, wbytes, slot_bytes);
  };
  const bool full = t.row_bytes == nv * 32 * 16;
#define DUCHESS_BULK(NVV)                                                          \
  case NVV:                                                                        \
    if (full) go(score_rows_bulk_kernel<BF16, NVV, true>);                         \
    else go(score_rows_bulk_kernel<BF16, NVV, false>);                             \
    break;
  switch (nv) {
    DUCHESS_BULK(1) DUCHESS_BULK(2) DUCHESS_BULK(4) DUCHESS_BULK(8) DUCHESS_BULK(12)
    DUCHESS_BULK(16) DUCHESS_BULK(20)
    default: return cudaErrorInvalidValue;
  }
#undef DUCHESS_BULK
  return cudaGetLastError();
}

template <bool BF16>
static cudaError_t launch_rows(const ScoreArgs& a, const TmaArgs& t, int nv, int grid,
                               cudaStream_t s) {
  const size_t wbytes = size_t(a.L) * a.H * sizeof(float);
  const bool wsmem = wbytes <= kRowsSmemMax;
  const size_t smem = wsmem ? wbytes : 0;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRowsWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a, t);
  };
#define DUCHESS_ROWS(NVV)                                                          \
  case NVV:                                                                        \
    if (wsmem) go(score_rows_kernel<BF16, NVV, true>);                             \
    else go(score_rows_kernel<BF16, NVV, false>);                                  \
    break;
  switch (nv) {
    DUCHESS_ROWS(1) DUCHESS_ROWS(2) DUCHESS_ROWS(4) DUCHESS_ROWS(8) DUCHESS_ROWS(12)
    DUCHESS_ROWS(16) DUCHESS_ROWS(20)
    default: return cudaErrorInvalidValue;
  }
#undef DUCHESS_ROWS
  return cudaGetLastError();
}

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Synthetic activation windows keyed by (seed, request, template, position).
template <bool BF16>
__global__ void __launch_bounds__(256) fill_kernel(char* acts, int64_t row_stride,
                                                   int64_t layer_stride, int64_t token_stride,
                                                   int L, int T, int H, uint64_t seed,
                                                   const int64_t* row_req, const int32_t* row_tmpl,
                                                   const int32_t* row_pos, const uint8_t* mask) {
  const int64_t unit = blockIdx.x;
  const int64_t row = unit / L;
  const int l = int(unit - row * L);
  if (mask != nullptr && mask[row] == 0) return;
  const uint64_t req = row_req ? uint64_t(row_req[row]) : uint64_t(row);
  const uint64_t tmpl = row_tmpl ? uint64_t(uint32_t(row_tmpl[row])) : 0ull;
  const uint64_t pos = row_pos ? uint64_t(uint32_t(row_pos[row])) : 0ull;
  const uint64_t rk = row_key(seed, req, tmpl, pos, uint64_t(l));
  const int64_t off = row * row_stride + int64_t(l) * layer_stride;
  const int64_t n = int64_t(T) * H;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int t = int(e / H), h = int(e - int64_t(t) * H);
    const float x = synth_value(rk, uint32_t(t), uint32_t(h));
    const int64_t idx = off + int64_t(t) * token_stride + h;
    if constexpr (BF16) reinterpret_cast<uint16_t*>(acts)[idx] = f32_to_bf16_rne(x);
    else reinterpret_cast<float*>(acts)[idx] = x;
  }
}

// Copy the listed rows of src (pinned host memory mapped into the device
// address space, or device memory) into the same rows of dst: only the
// survivors' windows cross PCIe. One CTA per listed row, 16-byte loads with
// 8 in flight per thread.
__global__ void __launch_bounds__(512) gather_rows_kernel(const char* src, char* dst,
                                                          int64_t row_bytes,
                                                          const int32_t* rows,
                                                          const int32_t* count,
                                                          const int32_t* par, int64_t stride) {
  int64_t n = *count;
  if (par) {
    const int p = *par;
    rows += p * stride;
    n = count[p];
  }
  const int64_t nv = row_bytes / 16;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t row = rows[i];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + row * row_bytes);
    uint4* d4 = reinterpret_cast<uint4*>(dst + row * row_bytes);
    for (int64_t v = threadIdx.x; v < nv; v += 8 * blockDim.x) {
      uint4 buf[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t j = v + int64_t(k) * blockDim.x;
        if (j < nv) buf[k] = __ldcg(s4 + j);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t j = v + int64_t(k) * blockDim.x;
        if (j < nv) __stcs(d4 + j, buf[k]);
      }
    }
  }
}

template <bool BF16, int NT>
static cudaError_t launch_fast(const ScoreArgs& a, int passes, cudaStream_t s) {
  const dim3 grid(unsigned(a.n_units * a.nsplit));
  switch (passes) {
    case 1: score_fast_kernel<BF16, NT, 1><<<grid, NT, 0, s>>>(a); break;
    case 2: score_fast_kernel<BF16, NT, 2><<<grid, NT, 0, s>>>(a); break;
    case 4: score_fast_kernel<BF16, NT, 4><<<grid, NT, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace duchess

using namespace duchess;

extern "C" size_t duchess_score_workspace_bytes(int64_t n_units, int32_t nsplit_max) {
  if (n_units <= 0 || nsplit_max <= 1) return 0;
  return size_t(n_units) * size_t(nsplit_max) * sizeof(float4) + size_t(n_units) * sizeof(unsigned);
}

static int score_impl(const void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                      int32_t T, int32_t H, int64_t row_stride, int64_t layer_stride,
                      int64_t token_stride, const float* wg, const float* c1,
                      const uint8_t* row_mask, const int32_t* row_list, const int32_t* row_count,
                      float* out_logit, double* out_prob, void* workspace, size_t workspace_bytes,
                      int32_t nsplit, int32_t threads, void* stream,
                      const int32_t* row_par = nullptr, int64_t list_stride = 0,
                      int32_t flags = 0) {
  if (n_rows < 0 || n_layers < 1 || T < 1 || H < 1) return DUCHESS_EINVAL;
  if (dtype != DUCHESS_F32 && dtype != DUCHESS_BF16) return DUCHESS_EINVAL;
  if (!acts || !wg || !c1 || !out_logit || !out_prob) return DUCHESS_EINVAL;
  if (n_rows == 0) return DUCHESS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool bf16 = dtype == DUCHESS_BF16;
  const int esz = bf16 ? 2 : 4, vec = 16 / esz;
  ScoreArgs a{};
  a.acts = static_cast<const char*>(acts);
  a.row_stride = row_stride;
  a.layer_stride = layer_stride;
  a.token_stride = token_stride;
  a.n_units = n_rows * n_layers;
  a.L = n_layers;
  a.T = T;
  a.H = H;
  a.wg = wg;
  a.c1 = c1;
  a.mask = row_mask;
  a.out_logit = out_logit;
  a.out_prob = out_prob;

  const bool aligned = (reinterpret_cast<uintptr_t>(acts) % 16 == 0) &&
                       ((row_stride * esz) % 16 == 0) && ((layer_stride * esz) % 16 == 0) &&
                       ((token_stride * esz) % 16 == 0) && (H % vec == 0) &&
                       (reinterpret_cast<uintptr_t>(wg) % 16 == 0);
  if (!aligned) {
    a.nsplit = 1;
    a.chunk = H;
    const size_t smem = size_t(H) * sizeof(float);
    if (smem > 200 * 1024) return DUCHESS_EINVAL;
    if (bf16) {
      cudaFuncSetAttribute(score_generic_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      score_generic_kernel<true><<<unsigned(a.n_units), 256, smem, s>>>(a);
    } else {
      cudaFuncSetAttribute(score_generic_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      score_generic_kernel<false><<<unsigned(a.n_units), 256, smem, s>>>(a);
    }
    return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
  }

  const int64_t row_bytes = int64_t(H) * esz;
  const bool tma_ok = row_bytes <= kTmaStageTarget * 4 && (row_bytes % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(acts) % 16 == 0);
  if (row_list && !(tma_ok && nsplit == 0 && threads == 0)) return DUCHESS_EINVAL;
  if (nsplit == 0 && threads == 0 && tma_ok) {
    TmaArgs t{};
    t.row_list = row_list;
    t.row_count = row_count;
    t.row_par = row_par;
    t.list_stride = list_stride;
    t.no_input_wait = (flags & DUCHESS_SCORE_NO_INPUT_WAIT) ? 1 : 0;
    t.row_bytes = int(row_bytes);
    t.contiguous = token_stride == H;
    // Tunables (env, for sweeps): CTAs per SM and stage size target.
    static const int cps = [] { const char* e = getenv("DUCHESS_K1_CPS"); int v = e ? atoi(e) : 2; return v < 1 ? 1 : (v > 4 ? 4 : v); }();
    // ~32 KB bulk copies (4 / 3 token rows at H = 4096 / 5120 bf16; three stages
    // per CTA at 2 CTAs/SM): C2 26.6-26.7 M branch-steps/s vs 26.1-26.2 with
    // ~20 KB copies and 0.95-0.98 of the copy peak with one row per copy; C3
    // 5.67-5.70 vs 5.58 M/s (DUCHESS_K1_STAGE sweeps)
    static const int stage_target = [] { const char* e = getenv("DUCHESS_K1_STAGE"); int v = e ? atoi(e) : kScoreStageTarget; return v < 4096 ? 4096 : v; }();
    const int nvec_row = int(row_bytes / 16);
    // 0: no warp-per-window kernel, 1: register pipeline, 2 (default): bulk-copy slots
    static const int rows_mode = [] { const char* e = getenv("DUCHESS_K1_ROWS"); return e ? atoi(e) : 2; }();
    // spill-free instantiations: bf16 rows up to 20 vectors per lane (H <= 5120),
    // fp32 up to 12 (H <= 1536); wider rows take the CTA kernel below
    if (rows_mode != 0 && T == 1 && nvec_row <= (bf16 ? 20 : 12) * 32 &&
        (reinterpret_cast<uintptr_t>(wg) % 16) == 0) {
      int nv = (nvec_row + 31) / 32;
      nv = nv <= 2 ? nv : nv <= 4 ? 4 : nv <= 8 ? 8 : (nv + 3) / 4 * 4;
      a.nsplit = 1;
      a.chunk = H;
      int slot_bytes = 0;
      const int64_t wbytes = (int64_t(H) * 4 + kBulkSlotAlign - 1) / kBulkSlotAlign * kBulkSlotAlign;
      const int bw = rows_mode == 2 && n_layers <= sm_count()
                         ? rows_bulk_warps(wbytes, row_bytes, 226 * 1024, slot_bytes) : 0;
      const int warps = bw >= 8 ? bw : kRowsWarps;
      int grid = sm_count();
      if (bw >= 8) {            // one probe layer per CTA: a multiple of L CTAs
        int64_t per_layer = grid / n_layers;
        if (!row_list && per_layer * warps > n_rows) per_layer = (n_rows + warps - 1) / warps;
        grid = int(per_layer * n_layers);
      } else if (!row_list && int64_t(grid) * warps > a.n_units) {
        grid = int((a.n_units + warps - 1) / warps);
      }
      cudaError_t e;
      if (bw >= 8)
        e = bf16 ? launch_rows_bulk<true>(a, t, nv, grid, bw, slot_bytes, s)
                 : launch_rows_bulk<false>(a, t, nv, grid, bw, slot_bytes, s);
      else
        e = bf16 ? launch_rows<true>(a, t, nv, grid, s) : launch_rows<false>(a, t, nv, grid, s);
      return e == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
    }
    t.tokens_per_stage = int(row_bytes >= stage_target ? 1 : stage_target / row_bytes);
    if (t.tokens_per_stage > T) t.tokens_per_stage = T;
    const int stage_bytes = t.tokens_per_stage * t.row_bytes;
    t.stages = (kTmaSmemBudget / cps) / stage_bytes;
    if (t.stages > 32) t.stages = 32;
    if (t.stages < 2) return DUCHESS_EINVAL;
    const int nvec = int(row_bytes / 16);
    int vpt = 1;
    while (vpt * kTmaCons < nvec) vpt <<= 1;
    if (vpt > 8) return DUCHESS_EINVAL;
    a.nsplit = 1;
    a.chunk = H;
    int grid = sm_count() * cps;
    if (!row_list && int64_t(grid) > a.n_units) grid = int(a.n_units);
    const cudaError_t e = bf16 ? launch_tma<true>(a, t, vpt, grid, s) : launch_tma<false>(a, t, vpt, grid, s);
    return e == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
  }
  int nt = threads > 0 ? threads : 256;
  if (nt != 128 && nt != 256 && nt != 512) return DUCHESS_EINVAL;
  const int cols_per_pass = nt * vec;
  const int passes_needed = (H + cols_per_pass - 1) / cols_per_pass;
  int ns = nsplit > 0 ? nsplit : (passes_needed + 1) / 2;
  if (ns > passes_needed) ns = passes_needed;
  int chunk = (H + ns - 1) / ns;
  chunk = (chunk + vec - 1) / vec * vec;
  int passes = (chunk + cols_per_pass - 1) / cols_per_pass;
  if (passes == 3) passes = 4;
  if (passes > 4) return DUCHESS_EINVAL;
  a.nsplit = ns;
  a.chunk = chunk;
  if (ns > 1) {
    if (workspace_bytes < duchess_score_workspace_bytes(a.n_units, ns) || !workspace)
      return DUCHESS_EINVAL;
    a.partials = static_cast<float4*>(workspace);
    a.counters = reinterpret_cast<unsigned*>(a.partials + a.n_units * ns);
  }
  cudaError_t e;
  if (bf16) {
    e = nt == 128 ? launch_fast<true, 128>(a, passes, s)
      : nt == 256 ? launch_fast<true, 256>(a, passes, s)
                  : launch_fast<true, 512>(a, passes, s);
  } else {
    e = nt == 128 ? launch_fast<false, 128>(a, passes, s)
      : nt == 256 ? launch_fast<false, 256>(a, passes, s)
                  : launch_fast<false, 512>(a, passes, s);
  }
  return e == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_score(const void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                             int32_t T, int32_t H, int64_t row_stride, int64_t layer_stride,
                             int64_t token_stride, const float* wg, const float* c1,
                             const uint8_t* row_mask, float* out_logit, double* out_prob,
                             void* workspace, size_t workspace_bytes, int32_t nsplit,
                             int32_t threads, void* stream) {
  return score_impl(acts, dtype, n_rows, n_layers, T, H, row_stride, layer_stride, token_stride,
                    wg, c1, row_mask, nullptr, nullptr, out_logit, out_prob, workspace,
                    workspace_bytes, nsplit, threads, stream);
}

extern "C" int duchess_score_list(const void* acts, int32_t dtype, int64_t n_rows,
                                  int32_t n_layers, int32_t T, int32_t H, int64_t row_stride,
                                  int64_t layer_stride, int64_t token_stride, const float* wg,
                                  const float* c1, const int32_t* row_list,
                                  const int32_t* row_count, float* out_logit, double* out_prob,
                                  void* stream) {
  if (!row_list || !row_count) return DUCHESS_EINVAL;
  return score_impl(acts, dtype, n_rows, n_layers, T, H, row_stride, layer_stride, token_stride,
                    wg, c1, nullptr, row_list, row_count, out_logit, out_prob, nullptr, 0, 0, 0,
                    stream);
}

extern "C" int duchess_fill_activations(void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                                        int32_t T, int32_t H, int64_t row_stride,
                                        int64_t layer_stride, int64_t token_stride, uint64_t seed,
                                        const int64_t* row_req, const int32_t* row_tmpl,
                                        const int32_t* row_pos, const uint8_t* row_mask,
                                        void* stream) {
  if (!acts || n_rows < 0 || n_layers < 1 || T < 1 || H < 1) return DUCHESS_EINVAL;
  if (n_rows == 0) return DUCHESS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned grid = unsigned(n_rows * n_layers);
  char* p = static_cast<char*>(acts);
  if (dtype == DUCHESS_BF16)
    fill_kernel<true><<<grid, 256, 0, s>>>(p, row_stride, layer_stride, token_stride, n_layers, T,
                                           H, seed, row_req, row_tmpl, row_pos, row_mask);
  else if (dtype == DUCHESS_F32)
    fill_kernel<false><<<grid, 256, 0, s>>>(p, row_stride, layer_stride, token_stride, n_layers, T,
                                            H, seed, row_req, row_tmpl, row_pos, row_mask);
  else
    return DUCHESS_EINVAL;
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_score_active_ex(const void* acts, int32_t dtype, int64_t n_rows,
                                       int32_t n_layers, int32_t T, int32_t H, int64_t row_stride,
                                       int64_t layer_stride, int64_t token_stride, const float* wg,
                                       const float* c1, const int32_t* active_rows,
                                       const int32_t* active_count, float* out_logit,
                                       double* out_prob, int32_t flags, void* stream) {
  if (!active_rows || !active_count) return DUCHESS_EINVAL;
  if (flags & ~DUCHESS_SCORE_NO_INPUT_WAIT) return DUCHESS_EINVAL;
  // DuchessState.active_count: [0..1] per-parity counts, [2] current parity
  return score_impl(acts, dtype, n_rows, n_layers, T, H, row_stride, layer_stride, token_stride,
                    wg, c1, nullptr, active_rows, active_count, out_logit, out_prob, nullptr, 0, 0,
                    0, stream, active_count + 2, n_rows, flags);
}

extern "C" int duchess_score_active(const void* acts, int32_t dtype, int64_t n_rows,
                                    int32_t n_layers, int32_t T, int32_t H, int64_t row_stride,
                                    int64_t layer_stride, int64_t token_stride, const float* wg,
                                    const float* c1, const int32_t* active_rows,
                                    const int32_t* active_count, float* out_logit,
                                    double* out_prob, void* stream) {
  return duchess_score_active_ex(acts, dtype, n_rows, n_layers, T, H, row_stride, layer_stride,
                                 token_stride, wg, c1, active_rows, active_count, out_logit,
                                 out_prob, 0, stream);
}

// DMA variant of the end-to-end input path: the caller holds the survivor
// rows on the host (e.g. read back with the round records); the rows are
// sorted, merged into runs of consecutive rows, and each run is one
// cudaMemcpyAsync from the host array into the same rows of dst, so the copy
// engines move the bytes (one large H2D DMA reaches ~55 GB/s on the box's
// link against ~51 GB/s for SM-initiated reads of the host mapping, and the
// two run side by side on different streams).
extern "C" int duchess_upload_rows(const void* src, void* dst, int64_t row_bytes,
                                   const int32_t* rows, int32_t n, int64_t n_rows, void* stream) {
  if (!src || !dst || row_bytes <= 0 || n < 0 || (n > 0 && !rows) || n_rows < 0)
    return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  std::vector<int32_t> r(rows, rows + n);
  std::sort(r.begin(), r.end());
  if (r.front() < 0 || r.back() >= n_rows) return DUCHESS_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  size_t i = 0;
  while (i < r.size()) {
    size_t j = i + 1;
    while (j < r.size() && r[j] <= r[j - 1] + 1) ++j;    // duplicates fold into the run
    const int64_t a = r[i], b = r[j - 1] + 1;
    if (cudaMemcpyAsync(d + a * row_bytes, s + a * row_bytes, size_t(b - a) * size_t(row_bytes),
                        cudaMemcpyHostToDevice, st) != cudaSuccess)
      return DUCHESS_ECUDA;
    i = j;
  }
  return DUCHESS_OK;
}

extern "C" int duchess_gather_active(const void* src, void* dst, int64_t row_bytes,
                                     const int32_t* active_rows, const int32_t* active_count,
                                     int64_t n_rows, void* stream) {
  if (!src || !dst || !active_rows || !active_count || row_bytes <= 0 || row_bytes % 16 ||
      n_rows < 0 || (reinterpret_cast<uintptr_t>(src) % 16) || (reinterpret_cast<uintptr_t>(dst) % 16))
    return DUCHESS_EINVAL;
  if (n_rows == 0) return DUCHESS_OK;
  const void* s = src;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, src) != cudaSuccess) {
    cudaGetLastError();
    return DUCHESS_EINVAL;
  }
  if (attr.type == cudaMemoryTypeUnregistered) return DUCHESS_EINVAL;   // pageable host memory
  if (attr.type == cudaMemoryTypeHost) {
    void* dp = nullptr;                          // pinned host memory: its device mapping
    if (cudaHostGetDevicePointer(&dp, const_cast<void*>(src), 0) != cudaSuccess) {
      cudaGetLastError();
      return DUCHESS_EINVAL;
    }
    s = dp;
  }
  gather_rows_kernel<<<sm_count() * 4, 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char*>(s), static_cast<char*>(dst), row_bytes, active_rows, active_count,
      active_count + 2, n_rows);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
