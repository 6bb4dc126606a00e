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
#include "kv_core.cuh"

namespace duchess {

__global__ void __launch_bounds__(kKvWarps * 32)
kv_round_kernel(DuchessPolicy pol, DuchessState s, DuchessKV kv) {
  extern __shared__ int32_t kv_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int r = blockIdx.x * (blockDim.x >> 5) + wib;
  // Overlapped launch (DUCHESS_KV_OVERLAP): this grid runs beside the
  // preceding kernel (the next round's scorer, which does not touch what is
  // read here) and waits for it only at the end, so the next duchess_round,
  // chained behind this grid, still sees the scorer's results.
  // Leading launch (DUCHESS_KV_LEAD): right after its duchess_round, which it
  // waits for; it then releases the next round's scorer at once (that scorer
  // streams beside it with DUCHESS_SCORE_NO_INPUT_WAIT and completes only
  // after it, so the next duchess_round sees the KV update done).
  const bool lead = kv.flags & DUCHESS_KV_LEAD;
  if (lead) pdl_wait();
  pdl_launch_dependents();
  if (r < s.n_slots) kv_slot_round(pol, s, kv, r, lane, kv_smem + int64_t(wib) * kv_warp_words(s.branch_cap));
  if (!lead) pdl_wait();
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
  attr[0].val.programmaticStreamSerializationAllowed =
      (kv->flags & (DUCHESS_KV_OVERLAP | DUCHESS_KV_LEAD)) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kv_round_kernel, *policy, *state, *kv);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

