// K4: fused logistic-regression gradient for probe training (one HBM pass).
//
// The reference ships no training ("OUT OF SCOPE ... training the
// MLPs"); the paper trains its probes with BCE. The
// north-star trains the linear probe of predictor.py:126-151 data-parallel:
//     g_h = inv_n * sum_i (sigmoid(x_i . w + b) - y_i) x_ih,   g_b = inv_n * sum_i (...)
// followed by an NCCL all-reduce of the H+1 gradient (python side).
//
// Blackwell design: one persistent CTA per SM; a producer warp streams row
// blocks into a shared-memory ring with cp.async.bulk (TMA bulk copies,
// completion tracked by mbarrier transaction counts). Default
// (lr_grad_split_kernel): eight "dot" warps compute each 64 KB stage's partial
// row dots and pass them through per-slot named barriers to eight "grad" warps,
// which form the residuals and accumulate residual * x into per-thread fp32
// registers from a second shared read of the stage; the two warp sets
// pipeline across stages (C5 on B200: 416 vs 350 M rows/s, 0.93 vs 0.78 of
// a read-only stream). Alternative (DUCHESS_K4_SPLIT=0, lr_grad_kernel):
// one warp set keeps a 32 KB stage's converted elements in registers and
// meets at one named barrier per stage. (Per-row mbarriers inside one warp
// set measured slower still: 0.74 vs 0.87 of the copy peak.) X is read from
// HBM exactly once. Per-CTA partial gradients are reduced in a fixed order by
// a second kernel (deterministic).
#include <cstdlib>

#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kConsWarps = 8;
constexpr int kCons = kConsWarps * 32;
constexpr int kStageBytesTarget = 32 * 1024;   // one warp set: two 16 KB rows fit the registers
constexpr int kStageBytesSplit = 64 * 1024;    // split dot / grad warps: fewer hand-offs per byte
constexpr int kMaxRB = 8;
constexpr int kKeepFloats = 128;   // g + w + kept stage per thread under 168 registers

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

template <int NTHREADS>
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory");
}

struct GradArgs {
  const char* X;
  const float* y;
  const float* w;
  int64_t n_rows;
  int H;
  int row_bytes;
  int rb;          // rows per stage
  int stages;
  int64_t rows_per_cta;
  float* partial;  // [grid, H+1]
};

// Row q's VPT vectors of this thread from the stage (zeros past the row end or
// past the stage's row count).
template <int NCONS, int VPT, bool FULL>
__device__ __forceinline__ void load_row(uint4 (&xv)[VPT], const char* base, int q, int nr,
                                         int row_bytes, int nvec) {
  const uint4* rowv = reinterpret_cast<const uint4*>(base + size_t(q) * row_bytes);
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int v = j * NCONS + int(threadIdx.x);
    xv[j] = (q < nr && (FULL || v < nvec)) ? rowv[v] : make_uint4(0u, 0u, 0u, 0u);
  }
}

// CW consumer warps + 1 producer warp. KEEP: the stage's vectors stay in
// registers from the dot pass to the r * x pass (one shared read per element);
// otherwise each pass re-reads them (fewer registers, more CTAs per SM).
template <bool BF16, int CW, int VPT, int RB, bool FULL, bool KEEP>
__device__ __forceinline__ void lr_grad_body(const GradArgs& a) {
  constexpr int NCONS = CW * 32;
  constexpr int EPV = BF16 ? 8 : 4;   // elements per 16-byte vector
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full_bar[16], empty_bar[16];
  __shared__ float red[2][CW][RB];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = int64_t(blockIdx.x) * a.rows_per_cta;
  const int64_t row1 = lmin(a.n_rows, row0 + a.rows_per_cta);
  const int64_t n_my = lmax(int64_t(0), row1 - row0);
  const int64_t n_iter = (n_my + a.rb - 1) / a.rb;
  const int stage_bytes = a.rb * a.row_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    // ---- producer: TMA bulk copies of row blocks into the ring ----
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < n_iter; ++it) {
        mbar_wait(&empty_bar[s], ph ^ 1u);
        const int64_t r = row0 + it * a.rb;
        const int nr = int(lmin(a.rb, row1 - r));
        const uint32_t bytes = uint32_t(nr) * uint32_t(a.row_bytes);
        mbar_expect_tx(&full_bar[s], bytes);
        bulk_g2s(smem + size_t(s) * stage_bytes, a.X + r * a.row_bytes, bytes, &full_bar[s], pol);
        if (++s == a.stages) { s = 0; ph ^= 1u; }
      }
    }
    return;
  }

  // ---- consumers ----
  const int nvec = a.row_bytes / 16;
  float g[VPT][EPV];
  float wv[VPT][EPV];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int v = j * NCONS + int(threadIdx.x);
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      g[j][e] = 0.f;
      const int col = v * EPV + e;
      wv[j][e] = (v < nvec && col < a.H) ? a.w[col] : 0.f;
    }
  }
  const float bias = a.w[a.H];
  float gb = 0.f;

  int s = 0;
  uint32_t ph = 0;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t r = row0 + it * a.rb;
    const int nr = int(lmin(a.rb, row1 - r));
    float yv[RB];                       // labels prefetched before the stage wait
#pragma unroll
    for (int q = 0; q < RB; ++q) yv[q] = q < nr ? __ldg(a.y + r + q) : 0.f;
    mbar_wait(&full_bar[s], ph);
    const char* base = smem + size_t(s) * stage_bytes;
    // A row's shared loads are all issued before the first use, and each
    // vector has its own accumulator pair, so the loads overlap and the FFMA2
    // chains stay short.
    // KEEP: the converted elements of the stage stay in registers for the
    // r * x pass (no second shared read or conversion).
    float xf[KEEP ? RB : 1][KEEP ? VPT : 1][EPV];
    float dots[RB], dots2[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      dots[q] = 0.f;
      dots2[q] = 0.f;
      uint4 xv[VPT];
      load_row<NCONS, VPT, FULL>(xv, base, q, nr, a.row_bytes, nvec);
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const uint32_t xw[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
        float xe[EPV];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (BF16) {
            xe[2 * e] = bf16lo(xw[e]);
            xe[2 * e + 1] = bf16hi(xw[e]);
          } else {
            xe[e] = __uint_as_float(xw[e]);
          }
        }
        float p0 = 0.f, p1 = 0.f;
#pragma unroll
        for (int e = 0; e < EPV; e += 2) ffma2(p0, p1, wv[j][e], wv[j][e + 1], xe[e], xe[e + 1]);
        dots[q] += p0;
        dots2[q] += p1;
        if constexpr (KEEP) {
#pragma unroll
          for (int e = 0; e < EPV; ++e) xf[KEEP ? q : 0][KEEP ? j : 0][e] = xe[e];
        }
      }
    }
    const int buf = int(it & 1);
    // The RB rows' warp sums in one butterfly: each of the first log2(RB)
    // levels halves the rows a lane carries (lane bit 4, 3, ... picks which
    // half it keeps), the remaining levels sum within lane groups, so the warp
    // does 5 shuffles for all RB rows instead of 5 per row. Row q's sum ends
    // in the lanes whose top log2(RB) bits equal q's bit-reversed index;
    // rows past nr carry zeros.
    float v[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) v[q] = dots[q] + dots2[q];
    int width = RB;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      if (width > 1) {
        const bool upper = lane & o;
#pragma unroll
        for (int h = 0; h < RB / 2; ++h) {
          if (2 * h >= width) break;
          const float keep = upper ? v[2 * h + 1] : v[2 * h];
          const float send = upper ? v[2 * h] : v[2 * h + 1];
          v[h] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        width >>= 1;
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      }
    }
    {
      // after the pairing levels lane l holds the row whose index bits are
      // (bit 4 of l) for the first level, (bit 3) for the second, ...
      constexpr int LB = RB == 1 ? 0 : RB == 2 ? 1 : RB == 4 ? 2 : 3;
      int q = 0;
#pragma unroll
      for (int b = 0; b < LB; ++b) q |= ((lane >> (4 - b)) & 1) << b;
      const bool writer = (lane & ((1 << (5 - LB)) - 1)) == 0;   // first lane of its group
      if (writer && q < nr) red[buf][warp][q] = v[0];
    }
    if constexpr (KEEP) {
      // the stage's bytes are all in registers: hand the slot back now
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    consumer_bar<NCONS>();
    // lane q computes row q's residual (fixed-order sum of the warp partials),
    // then every lane takes it by shuffle
    float mine = 0.f;
    if (lane < nr) {
      float z = bias;
#pragma unroll
      for (int k = 0; k < CW; ++k) z += red[buf][k][lane];
      float yl = 0.f;
#pragma unroll
      for (int q = 0; q < RB; ++q) yl = lane == q ? yv[q] : yl;
      mine = 1.0f / (1.0f + __expf(-z)) - yl;
    }
    float res[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      res[q] = __shfl_sync(0xffffffffu, mine, q);
      gb += res[q];                                  // res = 0 for q >= nr
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      uint4 xv[VPT];
      if constexpr (!KEEP) load_row<NCONS, VPT, FULL>(xv, base, q, nr, a.row_bytes, nvec);
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        float xe[EPV];
        if constexpr (KEEP) {
#pragma unroll
          for (int e = 0; e < EPV; ++e) xe[e] = xf[KEEP ? q : 0][KEEP ? j : 0][e];
        } else {
          const uint32_t xw[4] = {xv[j].x, xv[j].y, xv[j].z, xv[j].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if constexpr (BF16) {
              xe[2 * e] = bf16lo(xw[e]);
              xe[2 * e + 1] = bf16hi(xw[e]);
            } else {
              xe[e] = __uint_as_float(xw[e]);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < EPV; e += 2)
          ffma2(g[j][e], g[j][e + 1], res[q], res[q], xe[e], xe[e + 1]);
      }
    }
    if constexpr (!KEEP) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    if (++s == a.stages) { s = 0; ph ^= 1u; }
  }

  float* out = a.partial + int64_t(blockIdx.x) * (a.H + 1);
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int v = j * NCONS + int(threadIdx.x);
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const int col = v * EPV + e;
      if (v < nvec && col < a.H) out[col] = g[j][e];
    }
  }
  if (threadIdx.x == 0) out[a.H] = gb;
}

// Split roles: CW "dot" warps and CW "grad" warps share each stage. The dot
// warps compute the stage's partial row dots and hand them over through a
// named barrier per ring slot (bar.arrive by the dot warps, bar.sync by the
// grad warps; a second barrier per slot returns the dot buffer); the grad
// warps form the residuals and accumulate r * x from a second read of the
// same shared stage, then release it. The dot chain of stage s + 1 (loads,
// FFMA2, butterfly) runs while the grad warps still work on stage s, instead
// of every warp meeting at one barrier per stage; the price is a second shared
// read + bf16 conversion per element. The grad warps' arrival releases the
// stage (the dot warps are done with it once they handed its dots over).
// Named barriers: 1 + s (dots of ring slot s ready), kSplitWar + s (slot s's
// dots consumed); id 0 is __syncthreads.
constexpr int kSplitMaxStages = 7;
constexpr int kSplitWar = 1 + kSplitMaxStages;
template <int BASE>
__device__ __forceinline__ void named_sync(int s, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(BASE + s), "r"(n) : "memory");
}
template <int BASE>
__device__ __forceinline__ void named_arrive(int s, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(BASE + s), "r"(n) : "memory");
}

template <bool BF16, int CW, int VPT, int RB, bool FULL>
__device__ __forceinline__ void lr_grad_split_body(const GradArgs& a) {
  constexpr int NCONS = CW * 32;
  constexpr int EPV = BF16 ? 8 : 4;
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full_bar[kSplitMaxStages], empty_bar[kSplitMaxStages];
  __shared__ float red[kSplitMaxStages][CW][RB];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = int64_t(blockIdx.x) * a.rows_per_cta;
  const int64_t row1 = lmin(a.n_rows, row0 + a.rows_per_cta);
  const int64_t n_my = lmax(int64_t(0), row1 - row0);
  const int64_t n_iter = (n_my + a.rb - 1) / a.rb;
  const int stage_bytes = a.rb * a.row_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 2 * CW) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < n_iter; ++it) {
        mbar_wait(&empty_bar[s], ph ^ 1u);
        const int64_t r = row0 + it * a.rb;
        const int nr = int(lmin(a.rb, row1 - r));
        const uint32_t bytes = uint32_t(nr) * uint32_t(a.row_bytes);
        mbar_expect_tx(&full_bar[s], bytes);
        bulk_g2s(smem + size_t(s) * stage_bytes, a.X + r * a.row_bytes, bytes, &full_bar[s], pol);
        if (++s == a.stages) { s = 0; ph ^= 1u; }
      }
    }
    return;
  }

  const bool dot_role = warp < CW;
  const int tid = int(threadIdx.x) - (dot_role ? 0 : NCONS);   // column slot within the role
  const int rw = dot_role ? warp : warp - CW;
  const int nvec = a.row_bytes / 16;
  float acc[VPT][EPV];     // dot warps: w; grad warps: g
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int v = j * NCONS + tid;
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const int col = v * EPV + e;
      acc[j][e] = dot_role && v < nvec && col < a.H ? a.w[col] : 0.f;
    }
  }
  const float bias = a.w[a.H];
  float gb = 0.f;

  auto convert = [&](const uint4& x, float (&xe)[EPV]) {
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (BF16) {
        xe[2 * e] = bf16lo(xw[e]);
        xe[2 * e + 1] = bf16hi(xw[e]);
      } else {
        xe[e] = __uint_as_float(xw[e]);
      }
    }
  };
  auto load_vecs = [&](uint4 (&xv)[VPT], const char* base, int q, int nr) {
    const uint4* rowv = reinterpret_cast<const uint4*>(base + size_t(q) * a.row_bytes);
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int v = j * NCONS + tid;
      xv[j] = (q < nr && (FULL || v < nvec)) ? rowv[v] : make_uint4(0u, 0u, 0u, 0u);
    }
  };

  int s = 0;
  uint32_t ph = 0;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t r = row0 + it * a.rb;
    const int nr = int(lmin(a.rb, row1 - r));
    const char* base = smem + size_t(s) * stage_bytes;
    if (dot_role) {
      mbar_wait(&full_bar[s], ph);
      float v[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        uint4 xv[VPT];
        load_vecs(xv, base, q, nr);
        float p0 = 0.f, p1 = 0.f;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          float xe[EPV];
          convert(xv[j], xe);
#pragma unroll
          for (int e = 0; e < EPV; e += 2) ffma2(p0, p1, acc[j][e], acc[j][e + 1], xe[e], xe[e + 1]);
        }
        v[q] = p0 + p1;
      }
      // the RB rows' warp sums in one butterfly (see lr_grad_body)
      int width = RB;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        if (width > 1) {
          const bool upper = lane & o;
#pragma unroll
          for (int h = 0; h < RB / 2; ++h) {
            if (2 * h >= width) break;
            const float keep = upper ? v[2 * h + 1] : v[2 * h];
            const float send = upper ? v[2 * h] : v[2 * h + 1];
            v[h] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
          width >>= 1;
        } else {
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
      }
      constexpr int LB = RB == 1 ? 0 : RB == 2 ? 1 : RB == 4 ? 2 : 3;
      int q = 0;
#pragma unroll
      for (int b = 0; b < LB; ++b) q |= ((lane >> (4 - b)) & 1) << b;
      // red[s] hand-off by named barriers (producer arrive / consumer sync):
      // 1 + s orders these writes before the grad warps' reads, kSplitWar + s
      // the grad warps' reads of the previous lap before these writes
      if (it >= a.stages) named_sync<kSplitWar>(s, 2 * NCONS);
      if ((lane & ((1 << (5 - LB)) - 1)) == 0 && q < nr) red[s][rw][q] = v[0];
      named_arrive<1>(s, 2 * NCONS);
    } else {
      float yl = lane < nr ? __ldg(a.y + r + lane) : 0.f;
      named_sync<1>(s, 2 * NCONS);   // the dots of stage s
      mbar_wait(&full_bar[s], ph);   // (complete already) the stage's bytes, for this warp
      float mine = 0.f;
      if (lane < nr) {
        float z = bias;
#pragma unroll
        for (int k = 0; k < CW; ++k) z += red[s][k][lane];
        mine = 1.0f / (1.0f + __expf(-z)) - yl;
      }
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const float rq = __shfl_sync(0xffffffffu, mine, q);
        gb += rq;                                   // 0 for q >= nr
        uint4 xv[VPT];
        load_vecs(xv, base, q, nr);
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          float xe[EPV];
          convert(xv[j], xe);
#pragma unroll
          for (int e = 0; e < EPV; e += 2) ffma2(acc[j][e], acc[j][e + 1], rq, rq, xe[e], xe[e + 1]);
        }
      }
      if (it + a.stages < n_iter) named_arrive<kSplitWar>(s, 2 * NCONS);   // red[s] read
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    if (++s == a.stages) { s = 0; ph ^= 1u; }
  }
  if (dot_role) return;

  float* out = a.partial + int64_t(blockIdx.x) * (a.H + 1);
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int v = j * NCONS + tid;
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const int col = v * EPV + e;
      if (v < nvec && col < a.H) out[col] = acc[j][e];
    }
  }
  if (tid == 0) out[a.H] = gb;
}

template <bool BF16, int VPT, int RB, bool FULL>
__global__ void __launch_bounds__(2 * kCons + 32, 1) lr_grad_split_kernel(GradArgs a) {
  lr_grad_split_body<BF16, kConsWarps, VPT, RB, FULL>(a);
}

// Default: one CTA per SM (8 + 1 warps = 3 warps per SM sub-partition, so up
// to 168 registers), the stage's converted elements kept in registers between
// the two passes. Measured on B200 at H = 8192 bf16: 0.87 of HBM, against 0.78
// for two CTAs per SM that re-read the stage (<= 96 registers) and 0.75 for
// 16 consumer warps.
template <bool BF16, int VPT, int RB, bool FULL>
__global__ void __maxnreg__(168) lr_grad_kernel(GradArgs a) {
  lr_grad_body<BF16, kConsWarps, VPT, RB, FULL, true>(a);
}
// Rows too wide to keep a stage in registers (g and w alone take VPT * 16
// floats): re-read the stage for the r * x pass.
template <bool BF16, int VPT, int RB, bool FULL>
__global__ void __maxnreg__(168) lr_grad_kernel_reread(GradArgs a) {
  lr_grad_body<BF16, kConsWarps, VPT, RB, FULL, false>(a);
}

// Fixed-order reduction of per-CTA partials, scaled by inv_n.
__global__ void grad_reduce_kernel(const float* partial, int n_parts, int n, float inv_n,
                                   float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
  for (int k = 0; k < n_parts; ++k) acc += partial[int64_t(k) * n + i];
  out[i] = acc * inv_n;
}

__global__ void sgd_kernel(float* w, const float* g, int n, float lr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] -= lr * g[i];
}

template <bool BF16, int VPT, int RB, bool FULL>
static cudaError_t launch_grad_full(const GradArgs& a, int keep, int grid, size_t smem,
                                    cudaStream_t s) {
  if (keep == 2) {                       // split dot / grad warps
    auto k = lr_grad_split_kernel<BF16, VPT, RB, FULL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 2 * kCons + 32, smem, s>>>(a);
    return cudaGetLastError();
  }
  void (*k)(GradArgs) = lr_grad_kernel_reread<BF16, VPT, RB, FULL>;
  if constexpr (VPT * (BF16 ? 8 : 4) * (2 + RB) <= kKeepFloats) {
    if (keep == 1) k = lr_grad_kernel<BF16, VPT, RB, FULL>;
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<grid, kCons + 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool BF16, int VPT, int RB>
static cudaError_t launch_grad_rb(const GradArgs& a, int keep, int grid, size_t smem,
                                  cudaStream_t s) {
  return a.row_bytes == VPT * kCons * 16
             ? launch_grad_full<BF16, VPT, RB, true>(a, keep, grid, smem, s)
             : launch_grad_full<BF16, VPT, RB, false>(a, keep, grid, smem, s);
}

template <bool BF16, int VPT>
static cudaError_t launch_grad(const GradArgs& a, int keep, int grid, size_t smem,
                               cudaStream_t s) {
  switch (a.rb) {
    case 1: return launch_grad_rb<BF16, VPT, 1>(a, keep, grid, smem, s);
    case 2: return launch_grad_rb<BF16, VPT, 2>(a, keep, grid, smem, s);
    case 4: return launch_grad_rb<BF16, VPT, 4>(a, keep, grid, smem, s);
    default: return launch_grad_rb<BF16, VPT, 8>(a, keep, grid, smem, s);
  }
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace duchess

using namespace duchess;

extern "C" size_t duchess_lr_grad_workspace_bytes(int32_t H) {
  if (H < 1) return 0;
  return size_t(2 * num_sms()) * size_t(H + 1) * sizeof(float);
}

extern "C" int duchess_lr_grad(const void* X, int32_t dtype, const float* y, const float* w,
                               int64_t n_rows, int32_t H, float inv_n, float* grad_out,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (!X || !y || !w || !grad_out || n_rows < 0 || H < 1) return DUCHESS_EINVAL;
  if (dtype != DUCHESS_F32 && dtype != DUCHESS_BF16) return DUCHESS_EINVAL;
  const int esz = dtype == DUCHESS_BF16 ? 2 : 4;
  const int64_t row_bytes = int64_t(H) * esz;
  if (row_bytes % 16 != 0 || reinterpret_cast<uintptr_t>(X) % 16 != 0) return DUCHESS_EINVAL;
  const int nvec = int(row_bytes / 16);
  const int vpt_needed = (nvec + kCons - 1) / kCons;
  int vpt = 1;
  while (vpt < vpt_needed) vpt <<= 1;
  if (vpt > 8) return DUCHESS_EINVAL;
  // Tunables (env, for sweeps): stage bytes target, keep the stage in registers.
  static const int split = [] { const char* e = getenv("DUCHESS_K4_SPLIT"); return e ? atoi(e) : 1; }();
  static const int stage_target = [] { const char* e = getenv("DUCHESS_K4_STAGE"); int v = e ? atoi(e) : split ? kStageBytesSplit : kStageBytesTarget; return v < 1024 ? 1024 : v; }();
  static const int keep_mode = [] { const char* e = getenv("DUCHESS_K4_KEEP"); return e ? atoi(e) : -1; }();
  int rb = int(lmax(1, lmin(kMaxRB, stage_target / row_bytes)));
  rb = rb >= 8 ? 8 : rb >= 4 ? 4 : rb >= 2 ? 2 : 1;   // compile-time rows per stage
  // g, w and the kept stage: VPT * (16 / esz) * (2 + rb) floats per thread
  // 2: split dot / grad warps; 1: one warp set keeping the stage in registers; 0: re-read
  const int keep = split ? 2 : keep_mode != 0 && vpt * (16 / esz) * (2 + rb) <= kKeepFloats ? 1 : 0;
  const int grid = num_sms();          // one CTA per SM (3 warps per sub-partition)
  const int smem_budget = 200 * 1024;
  if (!workspace || workspace_bytes < size_t(grid) * size_t(H + 1) * sizeof(float))
    return DUCHESS_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GradArgs a{};
  a.X = static_cast<const char*>(X);
  a.y = y;
  a.w = w;
  a.n_rows = n_rows;
  a.H = H;
  a.row_bytes = int(row_bytes);
  a.rb = rb;
  const int stage_bytes = a.rb * a.row_bytes;
  a.stages = int(lmin(keep == 2 ? kSplitMaxStages : 16, lmax(2, smem_budget / stage_bytes)));
  if (int64_t(a.stages) * stage_bytes > smem_budget) return DUCHESS_EINVAL;
  a.rows_per_cta = (n_rows + grid - 1) / grid;
  a.partial = static_cast<float*>(workspace);
  const size_t smem = size_t(a.stages) * stage_bytes;
  cudaError_t e;
  const bool bf16 = dtype == DUCHESS_BF16;
  switch (vpt) {
    case 1: e = bf16 ? launch_grad<true, 1>(a, keep, grid, smem, s) : launch_grad<false, 1>(a, keep, grid, smem, s); break;
    case 2: e = bf16 ? launch_grad<true, 2>(a, keep, grid, smem, s) : launch_grad<false, 2>(a, keep, grid, smem, s); break;
    case 4: e = bf16 ? launch_grad<true, 4>(a, keep, grid, smem, s) : launch_grad<false, 4>(a, keep, grid, smem, s); break;
    default: e = bf16 ? launch_grad<true, 8>(a, keep, grid, smem, s) : launch_grad<false, 8>(a, keep, grid, smem, s); break;
  }
  if (e != cudaSuccess) return DUCHESS_ECUDA;
  const int n = H + 1;
  grad_reduce_kernel<<<(n + 255) / 256, 256, 0, s>>>(a.partial, grid, n, inv_n, grad_out);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_sgd_update(float* w, const float* grad, int32_t n, float lr, void* stream) {
  if (!w || !grad || n < 0) return DUCHESS_EINVAL;
  if (n == 0) return DUCHESS_OK;
  sgd_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(w, grad, n, lr);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" const char* duchess_version(void) { return "duchess_b200 0.1.0 sm_100a"; }

extern "C" int duchess_device_arch(void) {
#if defined(__CUDA_ARCH__)
  return __CUDA_ARCH__;
#else
  return 1000;
#endif
}
