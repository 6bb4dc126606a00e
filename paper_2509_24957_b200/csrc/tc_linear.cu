// Tensor-core linear layer with a fused per-column epilogue (tcgen05 + TMEM +
// TMA), sm_100a: the hidden layers of the reference's MLP forward
// (predictor.py:126-151) batched over M input rows. Used by the complexity
// (difficulty) classifier, 4096 -> 2048 -> 1024 -> 512 -> 5 with batch-norm
// and GeLU, which the reference evaluates one
// vector at a time in fp64.
//
//   pre[i, j] = ln_fold ? (X_i . W'_j) / sigma_i - (mu_i / sigma_i) S_j + C_j
//                       :  X_i . W_j + C_j
//   y[i, j]   = act(pre[i, j] * BS_j + BT_j)        (act: none / relu / gelu)
//
// With ln_fold the input LayerNorm (predictor.py:134-138) is folded into the
// first layer: W' = W diag(ln_gain), S = W' 1, C = W ln_bias + b; mu / sigma
// are the row's population mean / std (eps 1e-5). BS / BT fold the
// inference batch-norm (predictor.py:141-143). Output bf16 (next layer's
// input) row-major [M, N].
//
// Persistent: one CTA per SM walks (128-row, 256-column) output tiles in
// row-tile-major order; warp 0 TMA producer (A = X[128x64], B = W[256x64]
// bf16, 128B swizzle, 4-stage ring), warp 1 TMEM allocator + single-thread
// tcgen05.mma issuer (M128 N256 K16, fp32 accumulate, two 256-column
// accumulators so a tile's epilogue overlaps the next tile's MMAs), warps 2-5
// the epilogue (tcgen05.ld 32 columns at a time, fold, activation, bf16
// store). With ln_fold each tile sums its 1/n_col_tiles share of its rows for
// the LN statistics and the row tile's tiles combine the shares (fixed order).
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_pair.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {
namespace tcl {
using namespace tcpair;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int THREADS = 192;       // producer + MMA + 4 epilogue warps
constexpr int THREADS_EW8 = 320;   // producer + MMA + 8 epilogue warps (two per TMEM lane quarter)
// CTA pair (cta_group::2): a 256 x 256 tile per pair, each CTA holding its 128
// rows of A and half (128 columns) of B per stage, so a stage is 32 KB
template <int CG> struct Cfg {
  static constexpr int B_ROWS = BN / CG;                    // B rows this CTA loads
  static constexpr int STAGE = A_BYTES + B_ROWS * BK * 2;   // 48 / 32 KB
  static constexpr int NST = CG == 1 ? STAGES : 6;
  static constexpr int SMEM_BYTES = NST * STAGE + 1024;
};

struct Args {
  int64_t M;
  int K, N;
  int ln_fold, act;
  int G;               // groups (probe layers): independent GEMMs sharing the launch
  int a_interleaved;   // X rows: 1 = [M, G, K] (row-major over (row, group)), 0 = [G, M, K]
  int64_t n_rt;        // row tiles per group
  const uint16_t* X;
  const float* S;
  const float* C;
  const float* BS;
  const float* BT;
  uint16_t* out;
  int* hdr;            // ln_fold workspace: [0] launch epoch, [1] exit counter
  float2* stats;       // [M * n_col_tiles] partial (sum x, sum x^2)
  int* ready;          // [n_row_tiles] published partials, cumulative over launches
  int64_t n_units;
};

__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Work unit u -> (group, row tile, column tile), group-major then row-tile-major,
// so the column tiles of one (group, row tile) run together (A tile L2-hot).
struct Unit {
  int g, mt, nt;
};
__device__ __forceinline__ Unit unit_of(int64_t u, int64_t n_rt, int n_tiles) {
  const int64_t per_g = n_rt * n_tiles;
  Unit x;
  x.g = int(u / per_g);
  const int64_t rem = u - int64_t(x.g) * per_g;
  x.mt = int(rem / n_tiles);
  x.nt = int(rem - int64_t(x.mt) * n_tiles);
  return x;
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16, A/B bf16 K-major, D fp32, M=128, N=256.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                           (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Exact (erf-based) GeLU, predictor.py:106-110.
__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// LNF / ACT are compile-time (one instantiation per layer kind), so the
// epilogue evaluates only its own activation (no GeLU computed and discarded).
// CG = 2: CTA pairs (cluster of 2, cta_group::2). A unit is then a 256-row x
// 256-column tile: each CTA loads its 128 rows of A and 128 of the tile's 256
// B columns, both TMA loads signal the leader's stage barrier, the leader's
// single thread issues M256 N256 K16 MMAs reading both CTAs' shared memory,
// and each CTA's TMEM holds its 128 rows (the commit reaches both CTAs); the
// epilogue is per CTA as with CG = 1 and hands the accumulator back to the
// leader's MMA thread. Per CTA a stage is 32 KB instead of 48 KB for the same
// MMA work, so each SM moves a third less operand data per FLOP.
template <bool LNF, int ACT, int CG>
__global__ void __launch_bounds__(LNF ? THREADS : THREADS_EW8, 1)
linear_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
              Args a) {
  using CF = Cfg<CG>;
  // Epilogue warps: without the LN fold the epilogue is per column only, so
  // two warps share each TMEM lane quarter (one half of the tile's columns
  // each) and a short-K layer's BN + GeLU epilogue keeps up with its MMAs.
  constexpr int EW = LNF ? 4 : 8;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[CF::NST], empty_bar[CF::NST], tmem_full[2], tmem_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k_blocks = a.K / BK;
  const int n_tiles = a.N / BN;
  const int rank = CG == 2 ? int(cluster_rank()) : 0;
  const bool leader = rank == 0;
  // work-unit walk: one per CTA (CG = 1) or per pair (CG = 2)
  const int64_t u0 = CG == 2 ? int64_t(blockIdx.x >> 1) : int64_t(blockIdx.x);
  const int64_t ustep = CG == 2 ? int64_t(gridDim.x >> 1) : int64_t(gridDim.x);
  const int64_t n_rt_u = CG == 2 ? (a.n_rt + 1) / 2 : a.n_rt;     // unit row tiles
  const int64_t n_units = int64_t(a.G) * n_rt_u * n_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < CF::NST; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], EW * CG);    // the epilogue warps of every CTA of the unit
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync_all();       // the leader's barriers exist before any signal
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // PDL: the setup above (barriers, TMEM allocation) overlaps the previous
  // layer's tail; its output is read only after this point.
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t tmem = tmem_base;
  const int stamp = LNF ? a.hdr[0] + 1 : 0;

  if (warp == 0) {
    if (lane == 0) {                                   // ---- TMA producer ----
      int it = 0;
      for (int64_t u = u0; u < n_units; u += ustep) {
        const Unit w = unit_of(u, n_rt_u, n_tiles);
        const int m0 = (w.mt * CG + rank) * BM, n0 = w.g * a.N + w.nt * BN + rank * CF::B_ROWS;
        const int ay = a.a_interleaved ? w.g : m0, az = a.a_interleaved ? m0 : w.g;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % CF::NST;
          mbar_wait(&empty_bar[s], ((it / CF::NST) & 1) ^ 1u);
          char* st = smem + s * CF::STAGE;
          if constexpr (CG == 2) {
            const uint32_t lb = leader_addr(&full_bar[s]);
            if (leader) mbar_expect_tx(&full_bar[s], 2 * CF::STAGE);   // both CTAs' bytes
            tma_load_3d_pair(st, &map_a, kb * BK, ay, az, lb);
            tma_load_2d_pair(st + A_BYTES, &map_b, kb * BK, n0, lb);
          } else {
            mbar_expect_tx(&full_bar[s], CF::STAGE);
            tma_load_3d(st, &map_a, kb * BK, ay, az, &full_bar[s]);
            tma_load_2d(st + A_BYTES, &map_b, kb * BK, n0, &full_bar[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {                         // ---- MMA issuer ----
      int it = 0, i = 0;
      for (int64_t u = u0; u < n_units; u += ustep, ++i) {
        const int acc = i & 1;
        mbar_wait(&tmem_empty[acc], ((i >> 1) & 1) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % CF::NST;
          mbar_wait(&full_bar[s], (it / CF::NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const char* st = smem + s * CF::STAGE;
          const uint64_t da = desc_sw128(st), db = desc_sw128(st + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if constexpr (CG == 2) mma2(d, da + uint64_t(2 * k), db + uint64_t(2 * k), (kb | k) ? 1u : 0u);
            else mma(d, da + uint64_t(2 * k), db + uint64_t(2 * k), (kb | k) ? 1u : 0u);
          }
          if constexpr (CG == 2) commit2(&empty_bar[s]);
          else commit(&empty_bar[s]);
        }
        if constexpr (CG == 2) commit2(&tmem_full[acc]);
        else commit(&tmem_full[acc]);
      }
    }
  } else {
    // ---- epilogue: row = 32 * (warp % 4) + lane (TMEM lane quarter) ----
    const int q = warp & 3;
    constexpr int COLS = BN / (EW / 4);                     // columns per epilogue warp
    const int c_lo = EW == 8 ? ((warp - 2) >> 2) * COLS : 0;
    int i = 0;
    for (int64_t u = u0; u < n_units; u += ustep, ++i) {
      const Unit w = unit_of(u, n_rt_u, n_tiles);
      const int g = w.g, mt = w.mt * CG + rank, nt = w.nt;   // mt: this CTA's 128-row tile
      const bool tile = mt < a.n_rt;                          // (the pair's 2nd half may be past M)
      const int64_t row = int64_t(mt) * BM + 32 * q + lane;
      const int64_t grow = int64_t(g) * a.M + row;       // (group, row) index, group-major
      const int64_t xrow = a.a_interleaved ? row * a.G + g : grow;
      const int64_t gmt = int64_t(g) * a.n_rt + mt;
      float rsig = 1.f, shift = 0.f;
      if (LNF && tile) {                               // overlaps this tile's MMAs
        const int nv = a.K / 8;
        const int v_lo = int(int64_t(nt) * nv / n_tiles), v_hi = int(int64_t(nt + 1) * nv / n_tiles);
        float sx = 0.f, sxx = 0.f;
        if (row < a.M) {
          const uint4* rp = reinterpret_cast<const uint4*>(a.X + xrow * a.K);
          for (int v0 = v_lo; v0 < v_hi; v0 += 8) {
            uint4 buf[8];
#pragma unroll
            for (int w8 = 0; w8 < 8; ++w8) buf[w8] = v0 + w8 < v_hi ? __ldg(rp + v0 + w8) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int w8 = 0; w8 < 8; ++w8) {
              const uint32_t w4[4] = {buf[w8].x, buf[w8].y, buf[w8].z, buf[w8].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float lo = bf16lo(w4[e]), hi = bf16hi(w4[e]);
                sx += lo + hi;
                sxx = fmaf(lo, lo, fmaf(hi, hi, sxx));
              }
            }
          }
          a.stats[grow * n_tiles + nt] = make_float2(sx, sxx);
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          __threadfence();
          atomicAdd(a.ready + gmt, 1);
        }
        if (lane == 0)
          while (ld_acquire_s32(a.ready + gmt) < stamp * n_tiles) __nanosleep(64);
        __syncwarp();
        if (row < a.M) {
          float tx = 0.f, txx = 0.f;
          for (int t = 0; t < n_tiles; ++t) {
            const float2 p = __ldcg(a.stats + grow * n_tiles + t);
            tx += p.x;
            txx += p.y;
          }
          const float mean = tx / float(a.K);
          const float var = fmaxf(txx / float(a.K) - mean * mean, 0.f);
          rsig = rsqrtf(var + kLayerNormEps);
          shift = mean * rsig;
        }
      }
      const int acc = i & 1;
      mbar_wait(&tmem_full[acc], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * BN);
      const int n0 = nt * BN;
      const int64_t gp = int64_t(g) * a.N;               // group's per-column parameters
#pragma unroll 1
      for (int c0 = c_lo; c0 < c_lo + COLS; c0 += 32) {
        float v[32];
        tmem_ld32(base + uint32_t(c0), v);
        const int j0 = n0 + c0;
        const int64_t pj = gp + j0;
        uint32_t packed[16];
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          // per-column parameters of 4 columns at once (broadcast 16-byte loads)
          const float4 c4 = __ldg(reinterpret_cast<const float4*>(a.C + pj + k));
          const float4 bs4 = __ldg(reinterpret_cast<const float4*>(a.BS + pj + k));
          const float4 bt4 = __ldg(reinterpret_cast<const float4*>(a.BT + pj + k));
          float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (LNF) s4 = __ldg(reinterpret_cast<const float4*>(a.S + pj + k));
          const float cc[4] = {c4.x, c4.y, c4.z, c4.w}, bs[4] = {bs4.x, bs4.y, bs4.z, bs4.w};
          const float bt[4] = {bt4.x, bt4.y, bt4.z, bt4.w}, ss[4] = {s4.x, s4.y, s4.z, s4.w};
          float y[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            float pre = LNF ? fmaf(v[k + h], rsig, fmaf(-shift, ss[h], cc[h])) : v[k + h] + cc[h];
            pre = fmaf(pre, bs[h], bt[h]);
            y[h] = ACT == 1 ? fmaxf(pre, 0.f) : ACT == 2 ? gelu(pre) : pre;
          }
          packed[k / 2] = uint32_t(f32_to_bf16_rne(y[0])) | (uint32_t(f32_to_bf16_rne(y[1])) << 16);
          packed[k / 2 + 1] = uint32_t(f32_to_bf16_rne(y[2])) | (uint32_t(f32_to_bf16_rne(y[3])) << 16);
        }
        if (row < a.M) {
          uint4* dst = reinterpret_cast<uint4*>(a.out + grow * a.N + j0);
#pragma unroll
          for (int w = 0; w < 4; ++w)
            dst[w] = make_uint4(packed[4 * w], packed[4 * w + 1], packed[4 * w + 2], packed[4 * w + 3]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(leader_addr(&tmem_empty[acc]));
        else mbar_arrive(&tmem_empty[acc]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync_all();       // both CTAs done with the pair's TMEM
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (LNF && threadIdx.x == 0) {                     // last CTA out advances the epoch
    __threadfence();
    if (atomicAdd(a.hdr + 1, 1) == int(gridDim.x) - 1) {
      a.hdr[1] = 0;
      a.hdr[0] = stamp;
    }
  }
}

// Input LayerNorm normalisation (predictor.py:134-136) as its own pass: one
// CTA per row, fp64 sums (mean, then the centred square sum), writes
// z = (x - mean) / sqrt(var + 1e-5) as bf16. Feeding z (zero mean, unit scale)
// to the first tensor-core layer instead of folding the statistics into its
// epilogue avoids the cancellation of x.W' - mu * S for rows with a large
// common offset (the fold is exact algebra but not in fp32 / bf16).
template <typename TX>
__global__ void __launch_bounds__(256) row_normalize_kernel(const TX* X, int64_t M, int K,
                                                            uint16_t* Z) {
  __shared__ double red[8];
  const int64_t row = blockIdx.x;
  const TX* x = X + row * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto block_sum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    __syncthreads();
    return t;
  };
  double s = 0.0;
  for (int k = threadIdx.x; k < K; k += 256) s += double(x[k]);
  const double mean = block_sum(s) / K;
  double q = 0.0;
  for (int k = threadIdx.x; k < K; k += 256) {
    const double d = double(x[k]) - mean;
    q += d * d;
  }
  const double inv = 1.0 / sqrt(block_sum(q) / K + double(kLayerNormEps));
  for (int k = threadIdx.x; k < K; k += 256)
    Z[row * K + k] = f32_to_bf16_rne(float((double(x[k]) - mean) * inv));
}

// Vectorised variant for bf16 / fp32 rows with K % 8 == 0 and K <= 256 * 8 *
// RV: each thread loads its 8-element chunks once (16 B of bf16 or 32 B of
// fp32 per chunk) and keeps them in registers for the mean, the centred
// square sum (fp64 accumulation) and the normalised output, stored 16 B at a
// time.
template <bool BF16, int RV>
__global__ void __launch_bounds__(256) row_normalize_vec_kernel(const void* X, int64_t M, int K,
                                                                uint16_t* Z) {
  __shared__ double red[8];
  const int64_t row = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = K / 8;
  auto block_sum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    __syncthreads();
    return t;
  };
  float v[RV][8];
#pragma unroll
  for (int c = 0; c < RV; ++c) {
    const int ch = c * 256 + threadIdx.x;
    if (ch < nch) {
      if constexpr (BF16) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(X) + row * K) + ch);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) { v[c][2 * e] = bf16lo(w4[e]); v[c][2 * e + 1] = bf16hi(w4[e]); }
      } else {
        const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(X) + row * K) + 2 * ch;
        const float4 a = __ldg(p), b = __ldg(p + 1);
        v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
        v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[c][e] = 0.f;
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < RV; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) s += double(v[c][e]);
  const double mean = block_sum(s) / K;
  double q = 0.0;
#pragma unroll
  for (int c = 0; c < RV; ++c) {
    if (c * 256 + int(threadIdx.x) < nch) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double d = double(v[c][e]) - mean;
        q += d * d;
      }
    }
  }
  const double inv = 1.0 / sqrt(block_sum(q) / K + double(kLayerNormEps));
#pragma unroll
  for (int c = 0; c < RV; ++c) {
    const int ch = c * 256 + threadIdx.x;
    if (ch < nch) {
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        o[e] = uint32_t(f32_to_bf16_rne(float((double(v[c][2 * e]) - mean) * inv))) |
               (uint32_t(f32_to_bf16_rne(float((double(v[c][2 * e + 1]) - mean) * inv))) << 16);
      reinterpret_cast<uint4*>(Z + row * K)[ch] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// bf16 rows (K % 8 == 0, 16 B-aligned): one WARP per row, persistent, with
// the rows staged in shared memory. The CTA-per-row kernel above meets at four
// __syncthreads per row, so an SM had only ~8 rows' loads in flight and the
// pass ran at half the copy rate. Here each warp owns two row slots: while it
// normalises row i from one slot, ONE cp.async.bulk (lane 0, mbarrier
// transaction count) fills the other with its next row. Statistics: the mean
// from compensated fp32 sums per lane and fp64 across lanes, then d = (x - mean_hi) - mean_lo
// in fp32 with the mean split into two floats (no cancellation for rows with
// a large common offset), the centred square sum in fp32 per lane and fp64
// across lanes, z = d * inv rounded to bf16.
constexpr int kNormWarps = 4;

__global__ void __launch_bounds__(kNormWarps * 32) row_normalize_bulk_kernel(const uint16_t* X,
                                                                            int64_t M, int K,
                                                                            uint16_t* Z) {
  extern __shared__ __align__(128) unsigned char norm_smem[];
  __shared__ uint64_t bars[kNormWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t row_bytes = uint32_t(K) * 2u;
  const uint32_t slot_bytes = (row_bytes + 127u) & ~127u;
  unsigned char* slot0 = norm_smem + size_t(warp) * 2 * slot_bytes;
  const int64_t stride = int64_t(gridDim.x) * kNormWarps;
  int64_t row = int64_t(blockIdx.x) * kNormWarps + warp;
  if (lane == 0) {
    mbar_init(&bars[warp][0], 1);
    mbar_init(&bars[warp][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t pol = evict_first_policy();
  pdl_wait();                  // rows may come from the previous kernel
  pdl_launch_dependents();     // the first layer's setup may start on freed SMs
  if (lane == 0 && row < M) {
    mbar_expect_tx(&bars[warp][0], row_bytes);
    bulk_g2s(slot0, X + row * K, row_bytes, &bars[warp][0], pol);
  }
  const int nch = K / 8;
  for (int it = 0; row < M; ++it, row += stride) {
    const int b = it & 1;
    const uint4* sv = reinterpret_cast<const uint4*>(slot0 + size_t(b) * slot_bytes);
    if (lane == 0 && row + stride < M) {
      // the other slot was last read in iteration it - 1 (its reads completed
      // before the __syncwarp that ended it)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[warp][b ^ 1], row_bytes);
      bulk_g2s(slot0 + size_t(b ^ 1) * slot_bytes, X + (row + stride) * K, row_bytes,
               &bars[warp][b ^ 1], pol);
    }
    mbar_wait(&bars[warp][b], uint32_t(it >> 1) & 1u);
    // compensated fp32 sum per lane (TwoSum error terms accumulated apart;
    // error ~2^-46 of the sum of |x|, no fp64 conversion per element), then
    // fp64 across lanes
    float s0 = 0.f, c0 = 0.f, s1 = 0.f, c1 = 0.f;
    auto two_sum = [](float& s, float& c, float x) {
      const float t = s + x, bb = t - s;
      c += (s - (t - bb)) + (x - bb);
      s = t;
    };
    for (int ch = lane; ch < nch; ch += 32) {
      const uint4 u = sv[ch];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        two_sum(s0, c0, bf16lo(w4[e]));
        two_sum(s1, c1, bf16hi(w4[e]));
      }
    }
    double sm = (double(s0) + double(c0)) + (double(s1) + double(c1));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
    const double mean = sm / K;
    const float mh = float(mean), ml = float(mean - double(mh));
    float q0 = 0.f, q1 = 0.f;
    for (int ch = lane; ch < nch; ch += 32) {
      const uint4 u = sv[ch];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float d0 = (bf16lo(w4[e]) - mh) - ml, d1 = (bf16hi(w4[e]) - mh) - ml;
        q0 = fmaf(d0, d0, q0);
        q1 = fmaf(d1, d1, q1);
      }
    }
    double q = double(q0) + double(q1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = float(1.0 / sqrt(q / K + double(kLayerNormEps)));
    uint4* zr = reinterpret_cast<uint4*>(Z + row * K);
    for (int ch = lane; ch < nch; ch += 32) {
      const uint4 u = sv[ch];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        o[e] = pack_bf16x2_rn(((bf16lo(w4[e]) - mh) - ml) * inv, ((bf16hi(w4[e]) - mh) - ml) * inv);
      zr[ch] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    __syncwarp();
  }
}

// Classifier head (N small, e.g. 5): one warp per row, fp32 dots over the
// bf16 hidden vector, logits out.
__global__ void head_kernel(const uint16_t* Hm, int64_t M, int K, const float* W, const float* b,
                            int NO, float* logits) {
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const uint16_t* h = Hm + row * K;
  for (int o = 0; o < NO; ++o) {
    float acc = 0.f;
    for (int k = lane; k < K; k += 32) acc = fmaf(__uint_as_float(uint32_t(h[k]) << 16), W[int64_t(o) * K + k], acc);
    acc = warp_sum(acc);
    if (lane == 0) logits[row * NO + o] = acc + b[o];
  }
}

// Vector path (K % 8 == 0, K <= 256 * HC, aligned): a lane loads its 8-element
// chunks of the row once (16-byte loads), then forms every output's partial
// against the weight rows (float4 loads, L1-resident) and reduces per output.
template <int HC>
__global__ void head_vec_kernel(const uint16_t* Hm, int64_t M, int K, const float* W, const float* b,
                                int NO, float* logits) {
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int nch = K / 8;
  const uint4* h4 = reinterpret_cast<const uint4*>(Hm + row * K);
  uint4 hv[HC];
#pragma unroll
  for (int c = 0; c < HC; ++c) {
    const int ch = c * 32 + lane;
    hv[c] = ch < nch ? ldg_stream(h4 + ch) : make_uint4(0u, 0u, 0u, 0u);
  }
  for (int o = 0; o < NO; ++o) {
    const float4* w4 = reinterpret_cast<const float4*>(W + int64_t(o) * K);
    float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
    for (int c = 0; c < HC; ++c) {
      const int ch = c * 32 + lane;
      if (ch < nch) {
        const float4 wa = __ldg(w4 + 2 * ch), wb = __ldg(w4 + 2 * ch + 1);
        const uint32_t x[4] = {hv[c].x, hv[c].y, hv[c].z, hv[c].w};
        acc0 = fmaf(bf16lo(x[0]), wa.x, acc0);
        acc1 = fmaf(bf16hi(x[0]), wa.y, acc1);
        acc0 = fmaf(bf16lo(x[1]), wa.z, acc0);
        acc1 = fmaf(bf16hi(x[1]), wa.w, acc1);
        acc0 = fmaf(bf16lo(x[2]), wb.x, acc0);
        acc1 = fmaf(bf16hi(x[2]), wb.y, acc1);
        acc0 = fmaf(bf16lo(x[3]), wb.z, acc0);
        acc1 = fmaf(bf16hi(x[3]), wb.w, acc1);
      }
    }
    const float acc = warp_sum(acc0 + acc1);
    if (lane == 0) logits[row * NO + o] = acc + b[o];
  }
}

// Head with the weights in registers (NO outputs, K <= 256 * HC / 32 * 8):
// persistent warps, each lane holds its 8 * HC columns of every output row
// of W, so a row costs two 16-byte loads, NO * 8 * HC FMAs and NO warp sums
// (the vector kernel above re-loaded W for every row and output and ran at
// 1 TB/s on 33 MB). The next row's vectors are loaded before the current
// row's sums.
template <int NO, int HC>   // NO <= 8
__global__ void __launch_bounds__(256) head_reg_kernel(const uint16_t* Hm, int64_t M, int K,
                                                       const float* W, const float* b,
                                                       float* logits) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * (blockDim.x >> 5);
  int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nch = K / 8;
  float w[NO][HC][8];
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int c = 0; c < HC; ++c) {
      const int ch = c * 32 + lane;
#pragma unroll
      for (int e = 0; e < 8; ++e) w[o][c][e] = ch < nch ? W[int64_t(o) * K + ch * 8 + e] : 0.f;
    }
  float bias[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) bias[o] = b[o];
  pdl_wait();                  // the weights above overlap the last layer's tail
  pdl_launch_dependents();
  auto load = [&](int64_t r, uint4 (&hv)[HC]) {
    const uint4* h4 = reinterpret_cast<const uint4*>(Hm + r * K);
#pragma unroll
    for (int c = 0; c < HC; ++c) {
      const int ch = c * 32 + lane;
      hv[c] = r < M && ch < nch ? ldg_stream(h4 + ch) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  uint4 cur[HC];
  load(row, cur);
  for (; row < M; row += stride) {
    uint4 nxt[HC];
    load(row + stride, nxt);
    float acc[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) acc[o] = 0.f;
#pragma unroll
    for (int c = 0; c < HC; ++c) {
      const uint32_t x4[4] = {cur[c].x, cur[c].y, cur[c].z, cur[c].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = bf16lo(x4[e]), hi = bf16hi(x4[e]);
#pragma unroll
        for (int o = 0; o < NO; ++o) acc[o] = fmaf(hi, w[o][c][2 * e + 1], fmaf(lo, w[o][c][2 * e], acc[o]));
      }
    }
    // the NO warp sums in one transposed butterfly (8 value slots): each of the
    // first three levels halves the slots a lane carries (lane bit 4, 3, 2
    // picks the half), the last two sum within groups of four lanes — 9
    // shuffles instead of 5 per output
    float v[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) v[o] = o < NO ? acc[o < NO ? o : 0] : 0.f;
#pragma unroll
    for (int lvl = 0, width = 8; lvl < 3; ++lvl, width >>= 1) {
      const int off = 16 >> lvl;
      const bool upper = lane & off;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        if (2 * h >= width) break;
        const float keep = upper ? v[2 * h + 1] : v[2 * h];
        const float send = upper ? v[2 * h] : v[2 * h + 1];
        v[h] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int q = ((lane >> 4) & 1) | (((lane >> 3) & 1) << 1) | (((lane >> 2) & 1) << 2);
    float bq = 0.f;
#pragma unroll
    for (int o = 0; o < NO; ++o) bq = q == o ? bias[o] : bq;
    if ((lane & 3) == 0 && q < NO) logits[row * NO + q] = v[0] + bq;
#pragma unroll
    for (int c = 0; c < HC; ++c) cur[c] = nxt[c];
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// A operand: 3D map {K, Y, Z} of bf16 rows, box {BK, 1, BM} (interleaved
// [M, G, K]: Y = group, Z = row) or {BK, BM, 1} (group-major [G, M, K]).
static bool make_map_a(CUtensorMap* map, const void* base, uint64_t M, uint64_t G, uint64_t K,
                       bool interleaved) {
  auto enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {K, interleaved ? G : M, interleaved ? M : G};
  const cuuint64_t strides[2] = {K * 2, (interleaved ? G : M) * K * 2};
  const cuuint32_t box[3] = {uint32_t(BK), interleaved ? 1u : uint32_t(BM), interleaved ? uint32_t(BM) : 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {uint32_t(BK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tcl
}  // namespace duchess

using namespace duchess;

extern "C" size_t duchess_tc_linear_grouped_workspace_bytes(int64_t M, int32_t G, int32_t N) {
  if (M < 0 || G < 1 || N < tcl::BN) return 0;
  const int64_t mt = (M + tcl::BM - 1) / tcl::BM, nt = N / tcl::BN;
  return size_t(16 + int64_t(G) * M * nt * 8 + int64_t(G) * mt * 4 + 256);
}

extern "C" size_t duchess_tc_linear_workspace_bytes(int64_t M, int32_t N) {
  return duchess_tc_linear_grouped_workspace_bytes(M, 1, N);
}

extern "C" int duchess_tc_linear_grouped(const void* X, int64_t M, int32_t K, int32_t G,
                                         int32_t x_interleaved, const void* W, int32_t N,
                                         int32_t ln_fold, const float* S, const float* C,
                                         const float* BS, const float* BT, int32_t act, void* out,
                                         void* workspace, size_t workspace_bytes, void* stream) {
  if (!X || !W || !C || !BS || !BT || !out || (ln_fold && !S)) return DUCHESS_EINVAL;
  if (M < 0 || G < 1 || K < tcl::BK || K % tcl::BK || N < tcl::BN || N % tcl::BN || act < 0 ||
      act > 2)
    return DUCHESS_EINVAL;
  if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(W) % 16 ||
      reinterpret_cast<uintptr_t>(out) % 16 || reinterpret_cast<uintptr_t>(C) % 16 ||
      reinterpret_cast<uintptr_t>(BS) % 16 || reinterpret_cast<uintptr_t>(BT) % 16 ||
      (ln_fold && reinterpret_cast<uintptr_t>(S) % 16))      // per-column params read as float4
    return DUCHESS_EINVAL;
  if (ln_fold && (!workspace || workspace_bytes < duchess_tc_linear_grouped_workspace_bytes(M, G, N) ||
                  reinterpret_cast<uintptr_t>(workspace) % 16))
    return DUCHESS_EINVAL;
  if (M == 0) return DUCHESS_OK;
  // CTA pairs (cta_group::2) for K >= 1024 (measured faster: 2.01 -> 1.83 ms
  // for 5120 -> 2048 x 4 groups; with the 8-warp epilogue also for the
  // classifier's 2048 -> 1024 and 1024 -> 512 layers, 0.650 -> 0.641 ms per
  // batch), 1-CTA tiles for shorter K loops; DUCHESS_TC_PAIR=0 / 1 forces one
  // or the other (measurement)
  static const int pair_mode = [] { const char* e = getenv("DUCHESS_TC_PAIR"); return e ? atoi(e) : 2; }();
  const int CG = pair_mode == 2 ? (K >= 1024 ? 2 : 1) : (pair_mode ? 2 : 1);
  CUtensorMap ma, mb;
  if (!tcl::make_map_a(&ma, X, uint64_t(M), uint64_t(G), uint64_t(K), x_interleaved != 0))
    return DUCHESS_ECUDA;
  if (!tcl::make_map(&mb, W, uint64_t(G) * N, uint64_t(K), uint32_t(tcl::BN / CG)))
    return DUCHESS_ECUDA;
  const int64_t mt = (M + tcl::BM - 1) / tcl::BM, nt = N / tcl::BN;
  tcl::Args a{};
  a.M = M;
  a.K = K;
  a.N = N;
  a.G = G;
  a.a_interleaved = x_interleaved != 0;
  a.n_rt = mt;
  a.ln_fold = ln_fold;
  a.act = act;
  a.X = static_cast<const uint16_t*>(X);
  a.S = S;
  a.C = C;
  a.BS = BS;
  a.BT = BT;
  a.out = static_cast<uint16_t*>(out);
  if (ln_fold) {
    char* ws = static_cast<char*>(workspace);
    a.hdr = reinterpret_cast<int*>(ws);
    a.stats = reinterpret_cast<float2*>(ws + 16);
    a.ready = reinterpret_cast<int*>(ws + 16 + int64_t(G) * M * nt * 8);
  }
  a.n_units = int64_t(G) * ((mt + CG - 1) / CG) * nt;   // per CTA (CG 1) or per pair (CG 2)
  void (*kern)(CUtensorMap, CUtensorMap, tcl::Args);
  if (CG == 2)
    kern = ln_fold ? (act == 2 ? tcl::linear_kernel<true, 2, 2> : act == 1 ? tcl::linear_kernel<true, 1, 2>
                                                                           : tcl::linear_kernel<true, 0, 2>)
                   : (act == 2 ? tcl::linear_kernel<false, 2, 2> : act == 1 ? tcl::linear_kernel<false, 1, 2>
                                                                            : tcl::linear_kernel<false, 0, 2>);
  else
    kern = ln_fold ? (act == 2 ? tcl::linear_kernel<true, 2, 1> : act == 1 ? tcl::linear_kernel<true, 1, 1>
                                                                           : tcl::linear_kernel<true, 0, 1>)
                   : (act == 2 ? tcl::linear_kernel<false, 2, 1> : act == 1 ? tcl::linear_kernel<false, 1, 1>
                                                                            : tcl::linear_kernel<false, 0, 1>);
  const int smem = CG == 2 ? tcl::Cfg<2>::SMEM_BYTES : tcl::Cfg<1>::SMEM_BYTES;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one CTA per SM, all resident: with ln_fold tiles wait on statistics shares
  int64_t units_cap = CG == 2 ? sms / 2 : sms;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(CG * units_cap));
  cfg.blockDim = dim3(ln_fold ? tcl::THREADS : tcl::THREADS_EW8);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(CG);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (CG == 2) {
    // every pair must be resident at once (units wait on statistics other
    // CTAs publish): never launch more pairs than can be co-scheduled
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) == cudaSuccess && max_clusters > 0 &&
        max_clusters < units_cap)
      units_cap = max_clusters;
  }
  cfg.gridDim = dim3(unsigned(CG * (a.n_units < units_cap ? a.n_units : units_cap)));
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, a);
  return e == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_tc_linear(const void* X, int64_t M, int32_t K, const void* W, int32_t N,
                                 int32_t ln_fold, const float* S, const float* C, const float* BS,
                                 const float* BT, int32_t act, void* out, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  return duchess_tc_linear_grouped(X, M, K, 1, 0, W, N, ln_fold, S, C, BS, BT, act, out, workspace,
                                   workspace_bytes, stream);
}

extern "C" int duchess_row_normalize(const void* X, int32_t dtype, int64_t M, int32_t K, void* Z,
                                     void* stream) {
  if (!X || !Z || M < 0 || K < 1 ||
      (dtype != DUCHESS_F32 && dtype != DUCHESS_F64 && dtype != DUCHESS_BF16))
    return DUCHESS_EINVAL;
  if (M == 0) return DUCHESS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec = K % 8 == 0 && K <= 256 * 8 * 4 &&
                   (reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Z)) % 16 == 0;
  if (dtype == DUCHESS_BF16 && vec && K <= 8192) {   // one warp per row, rows staged in smem
    const size_t slot = (size_t(K) * 2 + 127) & ~size_t(127);
    const size_t smem = slot * 2 * tcl::kNormWarps;
    cudaFuncSetAttribute(tcl::row_normalize_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tcl::row_normalize_bulk_kernel,
                                                  tcl::kNormWarps * 32, smem);
    const int64_t need = (M + tcl::kNormWarps - 1) / tcl::kNormWarps;
    const unsigned grid = unsigned(need < int64_t(sms) * (per_sm < 1 ? 1 : per_sm)
                                       ? need : int64_t(sms) * (per_sm < 1 ? 1 : per_sm));
    tcl::row_normalize_bulk_kernel<<<grid, tcl::kNormWarps * 32, smem, st>>>(
        static_cast<const uint16_t*>(X), M, K, static_cast<uint16_t*>(Z));
    return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
  }
  if (dtype == DUCHESS_BF16 || (dtype == DUCHESS_F32 && vec)) {
    if (!vec) return DUCHESS_EINVAL;               // bf16 rows: vectorised path only
    const int rv = (K / 8 + 255) / 256;
    const bool bf = dtype == DUCHESS_BF16;
    if (rv <= 1) (bf ? tcl::row_normalize_vec_kernel<true, 1> : tcl::row_normalize_vec_kernel<false, 1>)
                     <<<unsigned(M), 256, 0, st>>>(X, M, K, static_cast<uint16_t*>(Z));
    else if (rv <= 2) (bf ? tcl::row_normalize_vec_kernel<true, 2> : tcl::row_normalize_vec_kernel<false, 2>)
                     <<<unsigned(M), 256, 0, st>>>(X, M, K, static_cast<uint16_t*>(Z));
    else (bf ? tcl::row_normalize_vec_kernel<true, 4> : tcl::row_normalize_vec_kernel<false, 4>)
             <<<unsigned(M), 256, 0, st>>>(X, M, K, static_cast<uint16_t*>(Z));
    return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
  }
  if (dtype == DUCHESS_F64)
    tcl::row_normalize_kernel<double><<<unsigned(M), 256, 0, st>>>(
        static_cast<const double*>(X), M, K, static_cast<uint16_t*>(Z));
  else
    tcl::row_normalize_kernel<float><<<unsigned(M), 256, 0, st>>>(
        static_cast<const float*>(X), M, K, static_cast<uint16_t*>(Z));
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_head_logits(const void* H, int64_t M, int32_t K, const float* W,
                                   const float* b, int32_t n_out, float* logits, void* stream) {
  if (!H || !W || !b || !logits || M < 0 || K < 1 || n_out < 1) return DUCHESS_EINVAL;
  if (M == 0) return DUCHESS_OK;
  const unsigned grid = unsigned((M + 7) / 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint16_t* h = static_cast<const uint16_t*>(H);
  const bool vec = K % 8 == 0 && reinterpret_cast<uintptr_t>(H) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(W) % 16 == 0 && K <= 256 * 8;
  if (vec && n_out == 5 && K <= 32 * 8 * 2) {      // the classifier's 5 levels
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tcl::head_reg_kernel<5, 2>, 256, 0);
    const int64_t cap = int64_t(sms) * (per_sm < 1 ? 1 : per_sm);
    const unsigned g = unsigned(int64_t(grid) < cap ? int64_t(grid) : cap);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tcl::head_reg_kernel<5, 2>, h, M, K, W, b, logits);
  } else if (vec && K <= 256 * 2) tcl::head_vec_kernel<2><<<grid, 256, 0, s>>>(h, M, K, W, b, n_out, logits);
  else if (vec) tcl::head_vec_kernel<8><<<grid, 256, 0, s>>>(h, M, K, W, b, n_out, logits);
  else tcl::head_kernel<<<grid, 256, 0, s>>>(h, M, K, W, b, n_out, logits);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
