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
// mean / std (eps 1e-5). One CTA per 128-row tile walks all hidden tiles of 256:
//   warp 0     TMA producer: A = X[128 x 64] and B = W1'[256 x 64] bf16 tiles
//              (128B swizzle) into a 4-stage shared-memory ring (mbarrier tx)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//              (M=128, N=256, K=16, fp32 accumulators in TMEM, double buffered
//              2 x 256 columns so the epilogue of tile j overlaps MMAs of j+1)
//   warps 2-5  row statistics (read from global while the first tile's MMAs
//              run), then the epilogue: tcgen05.ld 32 columns at a time, LN fold, bias,
//              ReLU, dot with w2 accumulated per row in registers.
// The hidden activations never touch HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kTcBM = 128, kTcBN = 256, kTcBK = 64, kTcStages = 4;
constexpr int kTcABytes = kTcBM * kTcBK * 2;            // 16 KB
constexpr int kTcBBytes = kTcBN * kTcBK * 2;            // 32 KB
constexpr int kTcStageBytes = kTcABytes + kTcBBytes;    // 48 KB
constexpr int kTcThreads = 192;                         // 6 warps
constexpr int kTcSmem = kTcStages * kTcStageBytes + 1024;  // + alignment slack

struct TcArgs {
  int64_t M;
  int K, NH;
  const float* s;
  const float* c;
  const float* w2;
  float b2;
  float* out_logit;
  double* out_prob;
  const uint16_t* X;   // row statistics are read straight from global (L2-hot)
};

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

__global__ void __launch_bounds__(kTcThreads, 1)
mlp_probe_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, TcArgs a) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[kTcStages], empty_bar[kTcStages];
  __shared__ uint64_t tmem_full[2], tmem_empty[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kTcBM;
  const int n_tiles = a.NH / kTcBN;
  const int k_blocks = a.K / kTcBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);          // MMA commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // 2 x 256 fp32 accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {   // ---- TMA producer ----
      int it = 0;
      for (int n = 0; n < n_tiles; ++n) {
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % kTcStages;
          const uint32_t ph = (it / kTcStages) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          char* st = smem + s * kTcStageBytes;
          mbar_expect_tx(&full_bar[s], kTcStageBytes);
          tma_load_2d(st, &map_a, kb * kTcBK, m0, &full_bar[s]);
          tma_load_2d(st + kTcABytes, &map_b, kb * kTcBK, n * kTcBN, &full_bar[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---- MMA issuer ----
      int it = 0;
      for (int n = 0; n < n_tiles; ++n) {
        const int acc = n & 1;
        mbar_wait(&tmem_empty[acc], ((n >> 1) & 1) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * kTcBN);
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % kTcStages;
          const uint32_t ph = (it / kTcStages) & 1;
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const char* st = smem + s * kTcStageBytes;
          const uint64_t da = umma_desc_sw128(st), db = umma_desc_sw128(st + kTcABytes);
#pragma unroll
          for (int k = 0; k < kTcBK / 16; ++k)   // +32 B per K=16 step inside the swizzle atom
            umma_bf16(d, da + uint64_t(2 * k), db + uint64_t(2 * k), (kb | k) ? 1u : 0u);
          umma_commit(&empty_bar[s]);
        }
        umma_commit(&tmem_full[acc]);
      }
    }
  } else {
    // ---- statistics + epilogue warps: row = 32 * (warp % 4) + lane (TMEM lane quarter) ----
    const int q = warp & 3;
    const int row_local = 32 * q + lane;
    const int64_t row = m0 + row_local;
    // Row statistics while the first hidden tile's MMAs run: 16-byte loads of the
    // row from global memory (the TMA producer streams the same rows, so they
    // are L2-resident), fp32 sums.
    float sx = 0.f, sxx = 0.f;
    if (row < a.M) {
      const uint4* rp = reinterpret_cast<const uint4*>(a.X + row * a.K);
      const int nv = a.K / 8;
      for (int v0 = 0; v0 < nv; v0 += 8) {
        uint4 buf[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) buf[u] = v0 + u < nv ? __ldg(rp + v0 + u) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t w4[4] = {buf[u].x, buf[u].y, buf[u].z, buf[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float lo = bf16lo(w4[e]), hi = bf16hi(w4[e]);
            sx += lo + hi;
            sxx = fmaf(lo, lo, fmaf(hi, hi, sxx));
          }
        }
      }
    }
    const float mean = sx / float(a.K);
    const float var = fmaxf(sxx / float(a.K) - mean * mean, 0.f);
    const float rsig = rsqrtf(var + kLayerNormEps);
    const float shift = mean * rsig;
    float logit = 0.f;
    for (int n = 0; n < n_tiles; ++n) {
      const int acc = n & 1;
      mbar_wait(&tmem_full[acc], (n >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + (uint32_t(32 * q) << 16) + uint32_t(acc * kTcBN);
#pragma unroll 1
      for (int c0 = 0; c0 < kTcBN; c0 += 32) {
        float v[32];
        tmem_ld32(base + uint32_t(c0), v);
        const int j0 = n * kTcBN + c0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float h = fmaf(v[i], rsig, fmaf(-shift, __ldg(a.s + j0 + i), __ldg(a.c + j0 + i)));
          logit = fmaf(fmaxf(h, 0.f), __ldg(a.w2 + j0 + i), logit);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
    }
    if (row < a.M) {
      const float z = logit + a.b2;
      a.out_logit[row] = z;
      double p = 1.0 / (1.0 + exp(-double(z)));
      a.out_prob[row] = fmin(fmax(p, kProbClip), 1.0 - kProbClip);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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

extern "C" int duchess_mlp_probe_tc(const void* X, int64_t M, int32_t K, const void* W1,
                                    int32_t NH, const float* s, const float* c, const float* w2,
                                    float b2, float* out_logit, double* out_prob, void* stream) {
  if (!X || !W1 || !s || !c || !w2 || !out_logit || !out_prob) return DUCHESS_EINVAL;
  if (M < 0 || K < kTcBK || K % kTcBK || NH < kTcBN || NH % kTcBN) return DUCHESS_EINVAL;
  if (reinterpret_cast<uintptr_t>(X) % 16 || reinterpret_cast<uintptr_t>(W1) % 16) return DUCHESS_EINVAL;
  if (M == 0) return DUCHESS_OK;
  CUtensorMap ma, mb;
  if (!make_map(&ma, X, uint64_t(M), uint64_t(K), kTcBM)) return DUCHESS_ECUDA;
  if (!make_map(&mb, W1, uint64_t(NH), uint64_t(K), kTcBN)) return DUCHESS_ECUDA;
  TcArgs a{M, K, NH, s, c, w2, b2, out_logit, out_prob, static_cast<const uint16_t*>(X)};
  cudaFuncSetAttribute(mlp_probe_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
  const unsigned grid = unsigned((M + kTcBM - 1) / kTcBM);
  mlp_probe_tc_kernel<<<grid, kTcThreads, kTcSmem, static_cast<cudaStream_t>(stream)>>>(ma, mb, a);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
