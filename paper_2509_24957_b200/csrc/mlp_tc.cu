// Tensor-core MLP probe (tcgen05 + TMEM + TMA), sm_100a.
//
// The paper's probe is an MLP on layer activations (reference
// predictor.py:126-151 evaluates it one vector at a time in fp64). Batched over
// N branch windows at T=1 it is a real GEMM (SURVEY §8(d) C3 variant,
// 5120 -> 2048 at ~2 kFLOP/B), so it runs on the 5th-gen tensor cores:
//
//   logit_i = b2 + sum_j w2_j * relu( (x_i . W1'_j - mu_i * s_j) / sigma_i + c_j )
//
// with W1' = W1 * diag(ln_gain) (bf16), s_j = sum_k W1'_jk, c_j = W1 ln_bias + b1
// (LayerNorm folded: predictor.py:134-140), mu_i / sigma_i the row's population
// mean / std (eps 1e-5).
//
// Persistent: one CTA per SM walks work units u = (row tile m, hidden tile h)
// of 128 rows x 256 hidden units in row-tile-major order (u += gridDim.x), so
// the grid is busy to within one unit (no 1.73-wave tail) and the 8 units of a
// row tile run at the same time on 8 CTAs (its A tiles stay L2-resident).
//   warp 0     TMA producer: A = X[128 x 64] and B = W1'[256 x 64] bf16 tiles
//              (128B swizzle) into a 4-stage shared-memory ring (mbarrier tx)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer (M=128,
//              N=256, K=16, fp32 in TMEM), accumulators double buffered across
//              units (2 x 256 columns) so unit i's epilogue overlaps unit i+1
//   warps 2-5  epilogue. Each unit sums its 1/n_tiles share of the row
//              tile's columns for the LN statistics (during its MMAs) and
//              publishes it; the units of a row tile combine the shares in
//              fixed order. Each unit reduces its 256 hidden columns to a
//              partial logit per row; the row tile's last unit sums the
//              partials in fixed hidden-tile order (deterministic).
// The hidden activations never touch HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "tc_pair.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kTcBM = 128, kTcBN = 256, kTcBK = 64, kTcStages = 4;
constexpr int kTcABytes = kTcBM * kTcBK * 2;            // 16 KB
constexpr int kTcThreads = 192;                         // 6 warps
// CTA pairs (cta_group::2, tc_pair.cuh): 256 x 256 units, each CTA loading its
// 128 rows of A and 128 of the unit's 256 hidden columns of B per 32 KB stage
template <int CG> struct TcCfg {
  static constexpr int B_ROWS = kTcBN / CG;
  static constexpr int STAGE = kTcABytes + B_ROWS * kTcBK * 2;
  static constexpr int NST = CG == 1 ? kTcStages : 6;
  static constexpr int SMEM_BYTES = NST * STAGE + 1024;
};

struct TcArgs {
  int64_t M;
  int K, NH;
  int G;               // groups (probe layers), each with its own W1 / s / c / w2 / b2
  int a_interleaved;   // X rows: 1 = [M, G, K], 0 = [G, M, K]
  int ln;              // 1 = LayerNorm folded into the GEMM (input layer), 0 = plain
  int64_t n_rt;        // row tiles per group
  const float* s;
  const float* c;
  const float* w2;
  const float* b2;     // [G]
  float* out_logit;    // [M, G]
  double* out_prob;    // [M, G]
  const uint16_t* X;   // row statistics are read straight from global (L2-hot)
  // workspace (zeroed once by the caller; kept consistent across launches)
  int* hdr;            // [0] launch epoch, [1] exit counter
  float2* stats;       // [M * n_tiles] per-unit partial (sum x, sum x^2) of the row
  float* partial;      // [M * n_tiles] partial logits
  int* ready;          // [n_row_tiles] published stat partials, cumulative over launches
  int* done;           // [n_row_tiles] finished hidden tiles
  int64_t n_units;     // n_row_tiles * n_tiles
};

__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void epi_bar() {   // the 4 epilogue warps
  asm volatile("bar.sync 2, 128;" ::: "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// unit -> (group, row tile, hidden tile), group-major then row-tile-major
__device__ __forceinline__ void tc_unit(int64_t u, int64_t n_rt, int n_tiles, int& g, int& mt, int& h) {
  const int64_t per_g = n_rt * n_tiles;
  g = int(u / per_g);
  const int64_t rem = u - int64_t(g) * per_g;
  mt = int(rem / n_tiles);
  h = int(rem - int64_t(mt) * n_tiles);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}

// Instruction descriptor: kind::f16, A/B bf16 K-major, D fp32, M=128, N=256.
constexpr uint32_t kTcIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kTcBN >> 3) << 17) |
                              (uint32_t(kTcBM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kTcIdesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
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

// CG = 2: on CTA pairs, as linear_kernel (tc_linear.cu): the leader issues the
// M256 N256 MMAs, both CTAs' TMA loads signal its stage barrier, each CTA's
// epilogue works on its own 128 rows and hands the accumulator back by a
// remote arrive on the leader's barrier.
template <int CG>
__global__ void __launch_bounds__(kTcThreads, 1)
mlp_probe_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, TcArgs a) {
  using namespace tcpair;
  using CF = TcCfg<CG>;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[CF::NST], empty_bar[CF::NST];
  __shared__ uint64_t tmem_full[2], tmem_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ int last_flag;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = a.NH / kTcBN;
  const int k_blocks = a.K / kTcBK;
  const int rank = CG == 2 ? int(cluster_rank()) : 0;
  const bool leader = rank == 0;
  const int64_t u0 = CG == 2 ? int64_t(blockIdx.x >> 1) : int64_t(blockIdx.x);
  const int64_t ustep = CG == 2 ? int64_t(gridDim.x >> 1) : int64_t(gridDim.x);
  const int64_t n_rt_u = CG == 2 ? (a.n_rt + 1) / 2 : a.n_rt;
  const int64_t n_units = int64_t(a.G) * n_rt_u * n_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < CF::NST; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);          // MMA commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 4 * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // 2 x 256 fp32 accumulator columns
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
  if constexpr (CG == 2) cluster_sync_all();
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const int stamp = a.hdr[0] + 1;          // this launch's "stats ready" stamp

  if (warp == 0) {
    if (lane == 0) {   // ---- TMA producer ----
      int it = 0;
      for (int64_t u = u0; u < n_units; u += ustep) {
        int g, mt, h;
        tc_unit(u, n_rt_u, n_tiles, g, mt, h);
        const int m0 = (mt * CG + rank) * kTcBM, n0 = g * a.NH + h * kTcBN + rank * CF::B_ROWS;
        const int ay = a.a_interleaved ? g : m0, az = a.a_interleaved ? m0 : g;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % CF::NST;
          const uint32_t ph = (it / CF::NST) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          char* st = smem + s * CF::STAGE;
          if constexpr (CG == 2) {
            const uint32_t lb = leader_addr(&full_bar[s]);
            if (leader) mbar_expect_tx(&full_bar[s], 2 * CF::STAGE);
            tma_load_3d_pair(st, &map_a, kb * kTcBK, ay, az, lb);
            tma_load_2d_pair(st + kTcABytes, &map_b, kb * kTcBK, n0, lb);
          } else {
            mbar_expect_tx(&full_bar[s], CF::STAGE);
            tma_load_3d(st, &map_a, kb * kTcBK, ay, az, &full_bar[s]);
            tma_load_2d(st + kTcABytes, &map_b, kb * kTcBK, n0, &full_bar[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {   // ---- MMA issuer ----
      int it = 0, i = 0;
      for (int64_t u = u0; u < n_units; u += ustep, ++i) {
        const int acc = i & 1;
        mbar_wait(&tmem_empty[acc], ((i >> 1) & 1) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * kTcBN);
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % CF::NST;
          const uint32_t ph = (it / CF::NST) & 1;
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const char* st = smem + s * CF::STAGE;
          const uint64_t da = umma_desc_sw128(st), db = umma_desc_sw128(st + kTcABytes);
#pragma unroll
          for (int k = 0; k < kTcBK / 16; ++k) {  // +32 B per K=16 step inside the swizzle atom
            if constexpr (CG == 2) mma2(d, da + uint64_t(2 * k), db + uint64_t(2 * k), (kb | k) ? 1u : 0u);
            else umma_bf16(d, da + uint64_t(2 * k), db + uint64_t(2 * k), (kb | k) ? 1u : 0u);
          }
          if constexpr (CG == 2) commit2(&empty_bar[s]);
          else umma_commit(&empty_bar[s]);
        }
        if constexpr (CG == 2) commit2(&tmem_full[acc]);
        else umma_commit(&tmem_full[acc]);
      }
    }
  } else {
    // ---- epilogue warps: row = 32 * (warp % 4) + lane (TMEM lane quarter) ----
    const int q = warp & 3;
    int i = 0;
    for (int64_t u = u0; u < n_units; u += ustep, ++i) {
      int g, mt, h;
      tc_unit(u, n_rt_u, n_tiles, g, mt, h);
      mt = mt * CG + rank;                           // this CTA's 128-row tile
      const bool tile = mt < a.n_rt;                 // (a pair's 2nd half may be past M)
      const int64_t row = int64_t(mt) * kTcBM + 32 * q + lane;
      const int64_t grow = int64_t(g) * a.M + row;          // (group, row), group-major
      const int64_t xrow = a.a_interleaved ? row * a.G + g : grow;
      const int64_t gmt = int64_t(g) * a.n_rt + mt;
      float rsig = 1.f, shift = 0.f;
      if (a.ln && tile) {
        // LN statistics: unit h sums its 1/n_tiles share of each row's columns
        // (while its MMAs run) and publishes the partial; every unit of the row
        // tile then combines the n_tiles partials in fixed order.
        const int nv = a.K / 8;
        const int v_lo = int(int64_t(h) * nv / n_tiles), v_hi = int(int64_t(h + 1) * nv / n_tiles);
        float sx = 0.f, sxx = 0.f;
        if (row < a.M) {
          const uint4* rp = reinterpret_cast<const uint4*>(a.X + xrow * a.K);
          for (int v0 = v_lo; v0 < v_hi; v0 += 8) {
            uint4 buf[8];
#pragma unroll
            for (int w = 0; w < 8; ++w) buf[w] = v0 + w < v_hi ? __ldg(rp + v0 + w) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int w = 0; w < 8; ++w) {
              const uint32_t w4[4] = {buf[w].x, buf[w].y, buf[w].z, buf[w].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float lo = bf16lo(w4[e]), hi = bf16hi(w4[e]);
                sx += lo + hi;
                sxx = fmaf(lo, lo, fmaf(hi, hi, sxx));
              }
            }
          }
          a.stats[grow * n_tiles + h] = make_float2(sx, sxx);
        }
        epi_bar();
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
      const uint32_t base = tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * kTcBN);
      // per-column parameters as broadcast float4 loads; four independent
      // partial logits (one per column residue mod 4), summed in fixed order
      float lg[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
      for (int c0 = 0; c0 < kTcBN; c0 += 32) {
        float v[32];
        tmem_ld32(base + uint32_t(c0), v);
        const int64_t j0 = int64_t(g) * a.NH + h * kTcBN + c0;   // group's column parameters
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 s4 = a.ln ? __ldg(reinterpret_cast<const float4*>(a.s + j0 + j))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 c4 = __ldg(reinterpret_cast<const float4*>(a.c + j0 + j));
          const float4 w4 = __ldg(reinterpret_cast<const float4*>(a.w2 + j0 + j));
          const float ss[4] = {s4.x, s4.y, s4.z, s4.w}, cc[4] = {c4.x, c4.y, c4.z, c4.w};
          const float ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float hv = fmaf(v[j + e], rsig, fmaf(-shift, ss[e], cc[e]));
            lg[e] = fmaf(fmaxf(hv, 0.f), ww[e], lg[e]);
          }
        }
      }
      const float logit = (lg[0] + lg[1]) + (lg[2] + lg[3]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(leader_addr(&tmem_empty[acc]));
        else mbar_arrive(&tmem_empty[acc]);
      }
      if (!tile) continue;
      if (row < a.M) a.partial[grow * n_tiles + h] = logit;
      // the row tile's last finished hidden tile sums the partials in fixed order
      epi_bar();
      if (threadIdx.x == 64) {
        __threadfence();
        last_flag = atomicAdd(a.done + gmt, 1) == n_tiles - 1;
      }
      epi_bar();
      if (last_flag) {
        __threadfence();
        if (row < a.M) {
          float z = a.b2[g];
          for (int t = 0; t < n_tiles; ++t) z += __ldcg(a.partial + grow * n_tiles + t);
          a.out_logit[row * a.G + g] = z;
          double p = 1.0 / (1.0 + exp(-double(z)));
          a.out_prob[row * a.G + g] = fmin(fmax(p, kProbClip), 1.0 - kProbClip);
        }
        if (threadIdx.x == 64) a.done[gmt] = 0;   // ready for the next launch
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (threadIdx.x == 0) {                        // last CTA out advances the epoch
    __threadfence();
    if (atomicAdd(a.hdr + 1, 1) == int(gridDim.x) - 1) {
      a.hdr[1] = 0;
      a.hdr[0] = stamp;
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

static bool make_map_a3(CUtensorMap* map, const void* base, uint64_t M, uint64_t G, uint64_t K,
                        bool interleaved) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {K, interleaved ? G : M, interleaved ? M : G};
  const cuuint64_t strides[2] = {K * 2, (interleaved ? G : M) * K * 2};
  const cuuint32_t box[3] = {uint32_t(kTcBK), interleaved ? 1u : uint32_t(kTcBM),
                             interleaved ? uint32_t(kTcBM) : 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {uint32_t(kTcBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace duchess

using namespace duchess;

extern "C" size_t duchess_mlp_probe_tc_grouped_workspace_bytes(int64_t M, int32_t G, int32_t NH) {
  if (M < 0 || G < 1 || NH < kTcBN) return 0;
  const int64_t mt = (M + kTcBM - 1) / kTcBM, nt = NH / kTcBN;
  return size_t(16 + int64_t(G) * M * nt * 8 + int64_t(G) * M * nt * 4 + 2 * int64_t(G) * mt * 4 + 256);
}

extern "C" size_t duchess_mlp_probe_tc_workspace_bytes(int64_t M, int32_t NH) {
  const size_t g = duchess_mlp_probe_tc_grouped_workspace_bytes(M, 1, NH);
  return g ? g + 32 : 0;                  // + the device copy of the scalar b2
}

extern "C" int duchess_mlp_probe_tc_grouped(const void* X, int64_t M, int32_t K, int32_t G,
                                            int32_t x_interleaved, int32_t ln, const void* W1,
                                            int32_t NH, const float* s, const float* c,
                                            const float* w2, const float* b2, float* out_logit,
                                            double* out_prob, void* workspace,
                                            size_t workspace_bytes, void* stream) {
  if (!X || !W1 || !c || !w2 || !b2 || !out_logit || !out_prob || (ln && !s)) return DUCHESS_EINVAL;
  if (M < 0 || G < 1 || K < kTcBK || K % kTcBK || NH < kTcBN || NH % kTcBN) return DUCHESS_EINVAL;
  if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(W1) % 16 ||
      (ln && reinterpret_cast<uintptr_t>(s) % 16) || reinterpret_cast<uintptr_t>(c) % 16 ||
      reinterpret_cast<uintptr_t>(w2) % 16)                     // per-column params read as float4
    return DUCHESS_EINVAL;
  if (!workspace || workspace_bytes < duchess_mlp_probe_tc_grouped_workspace_bytes(M, G, NH) ||
      reinterpret_cast<uintptr_t>(workspace) % 16)
    return DUCHESS_EINVAL;
  if (M == 0) return DUCHESS_OK;
  CUtensorMap ma, mb;
  if (!make_map_a3(&ma, X, uint64_t(M), uint64_t(G), uint64_t(K), x_interleaved != 0))
    return DUCHESS_ECUDA;
  // CTA pairs (cta_group::2) for long K loops (K >= 4096: measured faster, e.g.
  // 2.01 -> 1.83 ms for 5120 -> 2048 x 4 groups), 1-CTA tiles for short ones
  // (2048 -> 1024 x 4 groups: 347 vs 460 us with pairs); DUCHESS_TC_PAIR=0 / 1
  // forces one or the other (measurement)
  static const int pair_mode = [] { const char* e = getenv("DUCHESS_TC_PAIR"); return e ? atoi(e) : 2; }();
  const int CG = pair_mode == 2 ? (K >= 4096 ? 2 : 1) : (pair_mode ? 2 : 1);
  if (!make_map(&mb, W1, uint64_t(G) * NH, uint64_t(K), uint32_t(kTcBN / CG))) return DUCHESS_ECUDA;
  const int64_t mt = (M + kTcBM - 1) / kTcBM, nt = NH / kTcBN;
  char* ws = static_cast<char*>(workspace);
  TcArgs a{};
  a.M = M;
  a.K = K;
  a.NH = NH;
  a.G = G;
  a.a_interleaved = x_interleaved != 0;
  a.ln = ln != 0;
  a.n_rt = mt;
  a.s = s;
  a.c = c;
  a.w2 = w2;
  a.b2 = b2;
  a.out_logit = out_logit;
  a.out_prob = out_prob;
  a.X = static_cast<const uint16_t*>(X);
  a.hdr = reinterpret_cast<int*>(ws);
  a.stats = reinterpret_cast<float2*>(ws + 16);
  a.partial = reinterpret_cast<float*>(ws + 16 + int64_t(G) * M * nt * 8);
  a.ready = reinterpret_cast<int*>(ws + 16 + int64_t(G) * M * nt * 8 + int64_t(G) * M * nt * 4);
  a.done = a.ready + int64_t(G) * mt;
  a.n_units = int64_t(G) * ((mt + CG - 1) / CG) * nt;   // per CTA (CG 1) or per pair (CG 2)
  void (*kern)(CUtensorMap, CUtensorMap, TcArgs) =
      CG == 2 ? mlp_probe_tc_kernel<2> : mlp_probe_tc_kernel<1>;
  const int smem = CG == 2 ? TcCfg<2>::SMEM_BYTES : TcCfg<1>::SMEM_BYTES;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // every CTA resident (one per SM): units wait on statistics other CTAs publish
  int64_t units_cap = CG == 2 ? sms / 2 : sms;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(CG * units_cap));
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(CG);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
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

extern "C" int duchess_mlp_probe_tc(const void* X, int64_t M, int32_t K, const void* W1,
                                    int32_t NH, const float* s, const float* c, const float* w2,
                                    float b2, float* out_logit, double* out_prob,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  // one group, LayerNorm folded; the scalar b2 is staged after the grouped workspace
  const size_t gbytes = duchess_mlp_probe_tc_grouped_workspace_bytes(M, 1, NH);
  if (!workspace || gbytes == 0 || workspace_bytes < gbytes + 32) return DUCHESS_EINVAL;
  float* b2d = reinterpret_cast<float*>(static_cast<char*>(workspace) + (gbytes + 15) / 16 * 16);
  if (cudaMemcpyAsync(b2d, &b2, sizeof(float), cudaMemcpyHostToDevice,
                      static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return DUCHESS_ECUDA;
  return duchess_mlp_probe_tc_grouped(X, M, K, 1, 0, 1, W1, NH, s, c, w2, b2d, out_logit, out_prob,
                                      workspace, gbytes, stream);
}
