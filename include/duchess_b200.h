/* duchess_b200.h — C-ABI of the B200 DUCHESS probe + orchestration hot path.
 *
 * The reference (arxiv 2509.24957, `branchsim`, pure Python) has no FFI; its
 * seams for this path are Python callables. Each entry point below replaces
 * one of them, batched over many requests, and is what a ctypes / cffi binding
 * of the reference would call:
 *
 *   duchess_score            <- predictor.py:126-151  mlp_forward (linear probe),
 *                               called per survivor via the predictor seam
 *                               orchestrator.py:358-363; + token pooling (extension)
 *   duchess_advance          <- orchestrator.py:344-355  DuchessRun.step phase 1
 *                               (_decode_chunk :273-279, _probe :281-285, _collect :287-290)
 *                               + RequestRun.__init__ seeding :242-248 on refill
 *   duchess_decide           <- orchestrator.py:357-402  DuchessRun.step phases 2-5
 *                               (make_correctness_predictor :211-224, branch_out_sample
 *                               :188-197, _spawn :254-268, check_request_termination
 *                               :200-208, majority_vote core.py:76-83)
 *   duchess_sort_difficulty  <- scheduler.py:60-96  next_request pops over a snapshot
 *   duchess_fork_cow         <- orchestrator.py:254-268 _spawn(offset_base=source.position)
 *                               executed on a paged KV block table (extension)
 *   duchess_kv_round         <- the same forks (orchestrator.py:378-388) plus the
 *                               branches' decode / end / cancel lifecycle, applied every
 *                               round to a persistent paged KV cache (extension)
 *   duchess_lr_grad          <- probe training (absent in reference)
 *
 * Conventions: every pointer is caller-owned DEVICE memory unless stated;
 * every call is stream-ordered and non-blocking on `stream` (a cudaStream_t,
 * NULL = legacy default stream) and returns DUCHESS_OK (0) or an error code.
 * No C++ exception crosses this boundary.
 */
#ifndef DUCHESS_B200_H
#define DUCHESS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DUCHESS_F32 0
#define DUCHESS_BF16 1
#define DUCHESS_F64 2   /* row_normalize input only */

/* Branch status (orchestrator.py:35-40). */
#define DUCHESS_ACTIVE 0
#define DUCHESS_EARLY_TERMINATED 1
#define DUCHESS_NATURAL_END 2
#define DUCHESS_CAPPED 3
#define DUCHESS_CANCELLED 4

/* Request termination reasons (orchestrator.py:42-45). */
#define DUCHESS_REASON_NONE 0
#define DUCHESS_REASON_CONSENSUS 1
#define DUCHESS_REASON_COVERAGE 2
#define DUCHESS_REASON_EXHAUSTED 3

/* Branch actions (orchestrator.py:128-132). */
#define DUCHESS_ACT_CONTINUE 1
#define DUCHESS_ACT_TERMINATE 2
#define DUCHESS_ACT_BRANCH_OUT 3

/* Correctness-prediction source for DuchessRun.step phase 2. */
#define DUCHESS_PRED_DEVICE 0 /* probabilities from duchess_score (K1), by branch slot */
#define DUCHESS_PRED_TRACE 1  /* make_correctness_predictor: pred_probs else synthetic */
#define DUCHESS_PRED_HOST 2   /* caller-supplied probabilities by slot (predictor= callable) */

/* Policy flags. EXACT_CDF: always walk the branch-out CDF sequentially (the
 * default decides from a warp prefix sum unless u is within the rounding
 * margin of a boundary; both give identical picks — the flag exists to test that). */
#define DUCHESS_FLAG_EXACT_CDF 1

/* Policies (orchestrator.py:47-52). DUCHESS runs through advance / decide /
 * round; the baselines through duchess_baseline_round. */
#define DUCHESS_POLICY_DUCHESS 0
#define DUCHESS_POLICY_DEFAULT_SC 1
#define DUCHESS_POLICY_SHORT_MK 2
#define DUCHESS_POLICY_DYNASOR 3

#define DUCHESS_MT_WORDS 625 /* 624 MT19937 words + index, as random.Random.getstate() */
#define DUCHESS_MAX_SLOTS 64 /* max_branches limit of the warp-per-request kernel */
/* words per slot of the optional phase trace (DuchessState.trace) */
#define DUCHESS_TRACE_WORDS 24
#define DUCHESS_REC_WORDS 12

/* Round record fields (RoundReport, orchestrator.py:149-159, plus bookkeeping). */
#define DUCHESS_REC_ROUND 0     /* round_index; 0 = slot ran no round this step */
#define DUCHESS_REC_DECODING 1  /* decoding_branches */
#define DUCHESS_REC_MAX_CHUNK 2 /* max_chunk */
#define DUCHESS_REC_DECODE 3    /* decode_tokens */
#define DUCHESS_REC_PROBES 4    /* probes */
#define DUCHESS_REC_NACTIONS 5  /* len(actions) */
#define DUCHESS_REC_DONE 6      /* done */
#define DUCHESS_REC_NFORKS 7    /* branch_out actions this round */
#define DUCHESS_REC_NSURV 8     /* survivors scored + decided (branch-steps) */
#define DUCHESS_REC_REQ 9       /* pool index of the request in this slot */
#define DUCHESS_REC_REASON 10   /* termination reason if done */
#define DUCHESS_REC_FINAL 11    /* majority-vote answer id if done */

/* Counters (int64). */
#define DUCHESS_CNT_AMBIGUOUS 0 /* branch-out draws within 4 ulp of a CDF boundary */
#define DUCHESS_CNT_ERRORS 1    /* requests that hit "no answers collected" */
#define DUCHESS_CNT_FINISHED 2  /* requests finished */
#define DUCHESS_CNT_BRANCH_STEPS 3
#define DUCHESS_CNT_FORKS 4
#define DUCHESS_CNT_NEAR_TAU 5  /* PRED_DEVICE predictions within the probe tolerance of tau */
#define DUCHESS_N_COUNTERS 8

typedef struct DuchessPolicy {
  int32_t max_branches;      /* c, orchestrator.py:66 */
  int32_t interval_tokens;   /* i, :67 */
  int32_t early_term_rounds; /* S, :69 */
  int32_t token_cap;         /* :73 */
  int32_t probe_cost_tokens; /* :74 */
  int32_t need_consensus;    /* _at_least(consensus_frac, c), :162-164, :204 */
  int32_t need_coverage;     /* _at_least(coverage_frac, c), :206 */
  int32_t pred_source;       /* DUCHESS_PRED_* */
  int32_t n_layers;          /* probability columns per slot in `probs` */
  int32_t combine;           /* 0 = layer 0, 1 = mean over layers */
  int32_t flags;             /* DUCHESS_FLAG_* */
  int32_t policy_kind;       /* DUCHESS_POLICY_* (orchestrator.py:47-52) */
  int32_t short_m;           /* short-m@k m, :76 */
  int32_t dynasor_window;    /* dynasor D, :75 */
  int32_t _pad2[2];
  double early_term_threshold; /* tau, :68; +inf disables (:58-59) */
  double inv_temperature;      /* 1.0 / branch_out_temperature, computed by the host (:182) */
  double rho;                  /* SyntheticPredictorConfig.rho, predictor.py:321 */
} DuchessPolicy;

/* Read-only workload tables for a pool of P requests (workload.py:35-60).
 * Answers are interned per request in sorted string order with "" (NO_ANSWER)
 * as id 0, so min(id) == min(str) as majority_vote needs (core.py:83). */
typedef struct DuchessWorkload {
  int32_t n_requests;       /* P */
  int32_t queue_len;        /* entries in `queue` */
  int32_t cycle;            /* 1 = restart the queue when exhausted (steady-state bench) */
  int32_t _pad;
  const int32_t* tmpl_off;  /* [P+1] template CSR */
  const int32_t* ground_truth; /* [P] */
  const uint32_t* mt_init;  /* [P*625] random.Random(seed).getstate() */
  const int32_t* nat_len;   /* [NT] */
  const int32_t* final_ans; /* [NT] */
  const int32_t* conv;      /* [NT] oracle_convergence, -1 = None */
  const int32_t* probe_off; /* [NT+1] */
  const int32_t* probe_at;  /* [NP] */
  const int32_t* probe_ans; /* [NP] */
  const int32_t* pred_off;  /* [NT+1] */
  const int32_t* pred_at;   /* [NQ] */
  const double* pred_p;     /* [NQ] */
  const int32_t* queue;     /* [queue_len] pool indices in service order */
  const int32_t* queue_rec; /* [queue_len * 4] per queue position (pool index, template
                               base, template count, MT index word), 16-byte aligned, or
                               NULL: one load per refill instead of three */
} DuchessWorkload;

/* Mutable engine state: R request slots x C branch slots, Bmax branch ids. */
typedef struct DuchessState {
  int32_t n_slots;     /* R */
  int32_t branch_cap;  /* Bmax >= templates of any request */
  int32_t answer_cap;  /* A >= distinct answers of any request */
  int32_t _pad;
  /* per request slot [R] */
  int32_t* slot_req;
  int32_t* needs_refill;
  int32_t* n_branches;
  int32_t* next_template;
  int32_t* tokens_decode;
  int32_t* tokens_probe;
  int32_t* rounds;
  int32_t* done;
  int32_t* tally;      /* [R*A] */
  uint32_t* mt;        /* [R*625] */
  /* per branch [R*Bmax] */
  int32_t* br_offset;
  int32_t* br_decoded;
  int32_t* br_streak;
  int32_t* br_status;
  int32_t* br_final;
  int32_t* br_npred;
  int32_t* br_slot;
  double* br_last_pred;
  int32_t* br_probe_last; /* dynasor: last probed answer id (-1 none) */
  int32_t* br_probe_run;  /* dynasor: trailing run of identical probe answers */
  int32_t* slot_aux;      /* [R] short-m@k: finishers counted so far */
  /* per branch slot [R*C] */
  int32_t* slot_branch;
  uint8_t* row_mask;   /* survivors to score this round */
  int32_t* row_pos;
  int32_t* row_tmpl;
  int64_t* row_req;
  /* latest round */
  int32_t* p1_rec;     /* [R*8] phase-1 record of the round in flight (internal) */
  int32_t* round_rec;  /* [R*DUCHESS_REC_WORDS] latest completed round */
  int32_t* actions;    /* [R*2C*3] (kind, branch_id, source_branch_id or -1) */
  int32_t* forks;      /* [R*C*4]  (child, source, table_root, prefix_tokens) */
  double* step_pred;   /* [R*C] prediction used for each survivor, by slot */
  int32_t* queue_head; /* [2] */
  int32_t* active_rows;  /* [2*R*C] compacted survivor rows (r*C + slot) for K1 per list
                            parity, or NULL */
  int32_t* active_count; /* [8], 8-byte aligned: rows listed per parity [0..1], parity of
                            the list the next scorer reads [2], zero [3], duchess_round's
                            64-bit accumulator [4..5] (rows listed | slots done << 32),
                            zero [6..7] */
  /* outcomes by pool index [P] */
  int32_t* out_final;
  int32_t* out_reason;
  int32_t* out_tokens_decode;
  int32_t* out_tokens_probe;
  int32_t* out_rounds;
  int32_t* out_error;
  int32_t* out_tally;  /* [P*A] */
  long long* counters; /* [DUCHESS_N_COUNTERS] */
  long long* trace;    /* [R*DUCHESS_TRACE_WORDS] optional per-slot phase timestamps (ns), or NULL */
} DuchessState;

/* ---- K1: pooled LayerNorm + linear-probe scoring ------------------------ */
size_t duchess_score_workspace_bytes(int64_t n_units, int32_t nsplit_max);
int duchess_score(const void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers, int32_t T,
                  int32_t H, int64_t row_stride, int64_t layer_stride, int64_t token_stride,
                  const float* wg, const float* c1, const uint8_t* row_mask, float* out_logit,
                  double* out_prob, void* workspace, size_t workspace_bytes, int32_t nsplit,
                  int32_t threads, void* stream);
/* Same computation over a compacted device list of rows (row_list[0..*row_count),
 * e.g. DuchessState.active_rows written by duchess_advance): persistent,
 * TMA-bulk-staged kernel, one CTA per SM; n_rows bounds the row indices. */
int duchess_score_list(const void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                       int32_t T, int32_t H, int64_t row_stride, int64_t layer_stride,
                       int64_t token_stride, const float* wg, const float* c1,
                       const int32_t* row_list, const int32_t* row_count, float* out_logit,
                       double* out_prob, void* stream);
/* Score the survivors of an engine's round in flight: the list duchess_advance
 * / duchess_round left in DuchessState.active_rows / active_count (double
 * buffered; the parity word is read on the device). n_rows = R*C. */
int duchess_score_active(const void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                         int32_t T, int32_t H, int64_t row_stride, int64_t layer_stride,
                         int64_t token_stride, const float* wg, const float* c1,
                         const int32_t* active_rows, const int32_t* active_count,
                         float* out_logit, double* out_prob, void* stream);
/* duchess_score_active with flags: DUCHESS_SCORE_NO_INPUT_WAIT — the kernel
 * preceding this call in the stream does not produce its inputs (they were
 * final before that kernel started, e.g. duchess_kv_round with
 * DUCHESS_KV_LEAD right after the round that produced them): the scorer streams
 * without waiting for it (programmatic dependent launch) and still completes
 * only after it. */
#define DUCHESS_SCORE_NO_INPUT_WAIT 1
int duchess_score_active_ex(const void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                            int32_t T, int32_t H, int64_t row_stride, int64_t layer_stride,
                            int64_t token_stride, const float* wg, const float* c1,
                            const int32_t* active_rows, const int32_t* active_count,
                            float* out_logit, double* out_prob, int32_t flags, void* stream);
/* End-to-end input path: copy only the survivor rows (the engine's active list,
 * as duchess_score_active reads it) of an [n_rows, row_bytes] activation array
 * from src — pinned HOST memory (read over PCIe through its device mapping) or
 * device memory — into the same rows of the device array dst. */
int duchess_gather_active(const void* src, void* dst, int64_t row_bytes,
                          const int32_t* active_rows, const int32_t* active_count,
                          int64_t n_rows, void* stream);
/* The same copy by DMA for a survivor list the caller holds on the HOST (rows[n],
 * any order, each in [0, n_rows)): consecutive rows are merged into runs and
 * each run is one cudaMemcpyAsync (src pinned host memory, dst device) on
 * `stream`. */
int duchess_upload_rows(const void* src, void* dst, int64_t row_bytes, const int32_t* rows,
                        int32_t n, int64_t n_rows, void* stream);
int duchess_fill_activations(void* acts, int32_t dtype, int64_t n_rows, int32_t n_layers,
                             int32_t T, int32_t H, int64_t row_stride, int64_t layer_stride,
                             int64_t token_stride, uint64_t seed, const int64_t* row_req,
                             const int32_t* row_tmpl, const int32_t* row_pos,
                             const uint8_t* row_mask, void* stream);

/* ---- K2: per-request decisions (host pointers to the POD structs) -------- */
int duchess_advance(const DuchessPolicy* policy, const DuchessWorkload* workload,
                    const DuchessState* state, void* stream);
int duchess_decide(const DuchessPolicy* policy, const DuchessWorkload* workload,
                   const DuchessState* state, const double* probs, void* stream);

/* Round boundary: duchess_decide for the round in flight, then
 * duchess_advance for the next one, in one launch with no grid-wide barrier:
 * each slot is decided, refilled if it finished (the service queue is popped
 * atomically, so the requests admitted per round are those of decide +
 * advance; only their slot placement follows completion order) and advanced;
 * its survivors go to the other parity's active list, and the parity flips.
 * round_rec holds the round just decided. Needs active_rows / active_count. */
int duchess_round(const DuchessPolicy* policy, const DuchessWorkload* workload,
                  const DuchessState* state, const double* probs, void* stream);

/* One round of a baseline policy for every slot (DefaultScRun.step
 * orchestrator.py:408-435, ShortMkRun.step :466-516, DynasorRun.step
 * :529-561), refill included, in one launch: a slot whose request finished
 * pops the service queue atomically, then the policy round runs. Needs
 * active_count (the launch's exit count). No predictions, no forks. */
int duchess_baseline_round(const DuchessPolicy* policy, const DuchessWorkload* workload,
                           const DuchessState* state, void* stream);

/* Rule primitives (orchestrator.py:177-197, :200-208; core.py:76-83). */
int duchess_branch_out_sample(const double* probs, int32_t n, double inv_temperature,
                              uint32_t* mt_state, int32_t n_draws, int32_t* out_idx,
                              double* out_weights, long long* out_ambiguous, void* stream);
int duchess_vote(const int32_t* counts, int32_t n_sets, int32_t n_answers,
                 int32_t need_consensus, int32_t need_coverage, int32_t* out_final,
                 int32_t* out_reason, void* stream);
int duchess_template_lookup(const DuchessWorkload* workload, const int32_t* tmpl,
                            const int32_t* pos, int32_t n, int32_t* out_probe_answer,
                            double* out_trace_pred, void* stream);

/* synthetic_predict (predictor.py:328-335): n sequential draws from one
 * MT19937 stream (mt_state[625], updated in place). */
int duchess_synthetic_predict(uint32_t* mt_state, int32_t n, const int32_t* converged, double rho,
                              double* out, void* stream);
/* sample_confused_level (predictor.py:376-386); matrix is 5x5 row-major fp64. */
int duchess_confused_level(uint32_t* mt_state, int32_t n, const int32_t* true_level,
                           const double* matrix, int32_t* out, void* stream);
/* random.Random(seed) for n non-negative 64-bit seeds (CPython init_by_array
 * over the seed's 32-bit words) followed by the pending first twist: states
 * [n][625] with index 0 (the stream of random.Random(seed), pre-twisted). */
int duchess_mt_seed(const uint64_t* seeds, int32_t n, uint32_t* out_states, void* stream);
/* sample_confused_level for n requests, request i drawing once from its own
 * stream mt_states[i*625 .. +625) (simengine.py:223-227); states pre-twisted
 * (index <= 622, see engine.pretwist); read-only. */
int duchess_confused_levels(const uint32_t* mt_states, int32_t n, const int32_t* true_level,
                            const double* matrix, int32_t* out, void* stream);
/* run_simulation service timeline (simengine.py:247-257): for every slot whose
 * round record is live, service_ms[req] += round_time(decoding, max_chunk) +
 * probes * probe_cost_ms; first_token_ms[req] (init -1) := service_ms[req]
 * after the first round that decoded tokens. Indexed by pool request. */
int duchess_timeline(const int32_t* round_rec, int32_t n_slots, double ms_per_token,
                     double ms_per_extra_branch, int64_t probe_cost_ms, int64_t* service_ms,
                     int64_t* first_token_ms, void* stream);
/* check_early_termination (orchestrator.py:167-174) over CSR prediction histories. */
int duchess_early_termination(const double* history, const int32_t* offsets, int32_t n_sets,
                              double threshold, int32_t rounds, int32_t* out, void* stream);

/* ---- frozen MLP forward (predictor.py:126-151), fp64, any depth ----------
 * Packed parameters (fp64): [ln_gain H, ln_bias H] if has_ln, then per hidden
 * layer k: W_k [d_{k+1} x d_k] row-major, b_k, and if has_bn: mean, var,
 * gain, bias; then head W [head x d_last], b [head]. act[k]: 0 relu, 1 gelu.
 * Output per row: logits[head], probs[head] (clipped sigmoid if head == 1,
 * softmax otherwise). One CTA per input row. dims (n_hidden + 1 entries:
 * input and hidden widths) and act (n_hidden) are HOST arrays, passed by value;
 * params, x, logits, probs are device memory. */
int duchess_mlp_forward(const double* params, const int32_t* dims, int32_t n_hidden,
                        int32_t head_dim, const int32_t* act, int32_t has_ln, int32_t has_bn,
                        const double* x, int64_t n_rows, double* logits, double* probs,
                        void* stream);

/* ---- tensor-core MLP probe (tcgen05 + TMEM + TMA) -------------------------
 * logit_i = b2 + sum_j w2_j relu((X_i . W1g_j - mu_i s_j) / sigma_i + c_j):
 * the paper's MLP probe (one ReLU hidden layer, LayerNorm folded) batched as a
 * GEMM. X [M, K] bf16, W1g [NH, K] bf16 (K-major), s/c/w2 [NH] fp32;
 * K % 64 == 0, NH % 256 == 0. out_logit fp32 [M], out_prob fp64 [M]. */
size_t duchess_mlp_probe_tc_workspace_bytes(int64_t M, int32_t NH);
/* workspace: >= duchess_mlp_probe_tc_workspace_bytes(M, NH) bytes, 16-byte
 * aligned, ZEROED before its first use; the kernel keeps it reusable.
 * X, W1g, s, c, w2 16-byte aligned. */
int duchess_mlp_probe_tc(const void* X, int64_t M, int32_t K, const void* W1g, int32_t NH,
                         const float* s, const float* c, const float* w2, float b2,
                         float* out_logit, double* out_prob, void* workspace,
                         size_t workspace_bytes, void* stream);
/* Grouped form: G probes (one per probe layer) in one launch. X is [M, G, K]
 * (x_interleaved = 1: the engine's activation slab, one token per layer) or
 * [G, M, K] (0: e.g. the previous grouped layer's output); W1g [G*NH, K];
 * s/c/w2 [G*NH]; b2 [G] (device). ln = 0 skips the LayerNorm fold (a hidden
 * layer's input: pre = X.W1g_j + c_j). out_logit fp32 / out_prob fp64 [M, G].
 * The paper's probe LN -> 2048 -> 1024 -> 1 is
 * duchess_tc_linear_grouped (LN fold, ReLU) then this call with ln = 0. */
size_t duchess_mlp_probe_tc_grouped_workspace_bytes(int64_t M, int32_t G, int32_t NH);
int duchess_mlp_probe_tc_grouped(const void* X, int64_t M, int32_t K, int32_t G,
                                 int32_t x_interleaved, int32_t ln, const void* W1g, int32_t NH,
                                 const float* s, const float* c, const float* w2, const float* b2,
                                 float* out_logit, double* out_prob, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ---- tensor-core linear layer with fused epilogue (tcgen05 + TMEM + TMA) --
 * One hidden layer of mlp_forward (predictor.py:126-151) batched over M rows:
 * pre = ln_fold ? (X.W'_j)/sigma_i - (mu_i/sigma_i) S_j + C_j : X.W_j + C_j,
 * out = act(pre * BS_j + BT_j) as bf16 [M, N] (act 0 none, 1 relu, 2 gelu).
 * X [M, K] bf16, W [N, K] bf16 (K-major); K % 64 == 0, N % 256 == 0; X, W, out,
 * S, C, BS, BT 16-byte aligned. With
 * ln_fold the input LayerNorm is folded in (W' = W diag(gain), S = W' 1,
 * C = W ln_bias + b; row mean / std computed on the device). */
size_t duchess_tc_linear_workspace_bytes(int64_t M, int32_t N);
/* workspace (ln_fold only; may be NULL otherwise): >= the queried bytes,
 * 16-byte aligned, zeroed before first use, reusable afterwards. */
int duchess_tc_linear(const void* X, int64_t M, int32_t K, const void* W, int32_t N,
                      int32_t ln_fold, const float* S, const float* C, const float* BS,
                      const float* BT, int32_t act, void* out, void* workspace,
                      size_t workspace_bytes, void* stream);
/* Grouped form: G independent layers in one launch (one per probe layer). X
 * [M, G, K] (x_interleaved = 1) or [G, M, K] (0); W [G*N, K]; S/C/BS/BT [G*N];
 * out bf16 [G, M, N] (group-major). */
size_t duchess_tc_linear_grouped_workspace_bytes(int64_t M, int32_t G, int32_t N);
int duchess_tc_linear_grouped(const void* X, int64_t M, int32_t K, int32_t G,
                              int32_t x_interleaved, const void* W, int32_t N, int32_t ln_fold,
                              const float* S, const float* C, const float* BS, const float* BT,
                              int32_t act, void* out, void* workspace, size_t workspace_bytes,
                              void* stream);
/* Input LayerNorm as a pass: Z (bf16 [M, K]) = (X - mean) / sqrt(var + 1e-5)
 * per row of X ([M, K], DUCHESS_F32, DUCHESS_F64 or DUCHESS_BF16 — bf16 needs
 * K % 8 == 0, K <= 8192 and 16-byte aligned rows), statistics in fp64 (bf16
 * rows: compensated fp32 sums per lane, fp64 across lanes; the mean is split
 * into two floats for the centring) (predictor.py:134-136). */
int duchess_row_normalize(const void* X, int32_t dtype, int64_t M, int32_t K, void* Z,
                          void* stream);
/* Small classifier head: logits[M, n_out] = H (bf16 [M, K]) . W^T (fp32 [n_out, K]) + b. */
int duchess_head_logits(const void* H, int64_t M, int32_t K, const float* W, const float* b,
                        int32_t n_out, float* logits, void* stream);

/* ---- difficulty ordering (scheduler.py:60-96) --------------------------- */
int duchess_sort_difficulty(const uint64_t* keys, const int32_t* seg_offsets, int32_t n_segs,
                            int32_t* out_perm, void* stream);
/* The whole snapshot as one sequence (any n): out_perm = the permutation
 * sorting (key, index) ascending — 4096-key tiles sorted in shared memory,
 * then merge-path merge passes (device only; workspace from
 * duchess_sort_keys_workspace_bytes(n)). */
size_t duchess_sort_keys_workspace_bytes(int64_t n);
int duchess_sort_keys(const uint64_t* keys, int64_t n, int32_t* out_perm, void* workspace,
                      size_t workspace_bytes, void* stream);

/* ---- K3: copy-on-write block-table fork ----------------------------------
 * Fork records are (child, source, table_root, prefix_tokens) int32 quads laid
 * out as [n_groups][group_cap]; group g holds group_counts[g*counts_stride]
 * valid records (group_counts NULL: group_cap each). Branch ids map to block-
 * table rows g*rows_per_group + id. Forks are applied in (group, record)
 * order: the child row receives the root's first prefix/block_tokens entries
 * (refcount += 1 each); a partial tail block is taken from
 * free_list[*free_cursor + k] (k = rank among tail-needing forks), gets
 * refcount 1 and a copy of the root's first prefix%block_tokens tokens of KV
 * bytes. Remaining child entries are set to -1. *free_cursor advances by the
 * number of tail blocks taken. status[0] is set to 1 if the free list ran out. */
size_t duchess_fork_workspace_bytes(int32_t n_groups, int32_t group_cap);
int duchess_fork_cow(const int32_t* forks, int32_t group_cap, const int32_t* group_counts,
                     int32_t counts_stride, int32_t n_groups, int32_t rows_per_group,
                     int32_t* block_table, int32_t table_stride, int32_t* refcount,
                     const int32_t* free_list, int32_t free_list_len, int32_t* free_cursor,
                     void* kv_pool, int64_t kv_bytes_per_token, int32_t block_tokens,
                     int32_t* status, void* workspace, size_t workspace_bytes, void* stream);

/* ---- K3 in the round: persistent paged KV cache ---------------------------
 * Block tables for every branch of every request slot ([R*Bmax] rows of
 * max_blocks entries, global block ids, -1 = none). Slot r owns the arena of
 * blocks [r*P, (r+1)*P) (P = blocks_per_slot) with a LIFO free stack and a
 * high-water mark; the KV bytes of block b live at kv_pool + b * block_tokens *
 * kv_bytes_per_token (kv_pool may be NULL: tables only). arena[r*4 + k]: k = 0
 * stack top, 1 high-water mark, 2 owning pool index (-1 none), 3 peak blocks.
 * All arrays zero-initialised except table (-1) and arena[r*4+2] (-1). */
#define DUCHESS_KV_CNT_ALLOC 0       /* blocks allocated (appends + fork tails) */
#define DUCHESS_KV_CNT_FREE 1        /* blocks returned (refcount 0, arena resets) */
#define DUCHESS_KV_CNT_TAIL_BYTES 2  /* KV bytes copied for fork tails */
#define DUCHESS_KV_CNT_OVERFLOW 3    /* blocks that did not fit the arena / table */
#define DUCHESS_KV_N_COUNTERS 4
/* Launch overlapped with the preceding kernel in the stream (programmatic
 * dependent launch): the call runs while that kernel still runs and completes
 * only after it. Legal when the preceding kernel does not write the engine
 * state read here and releases its dependents only after its own inputs are
 * final — e.g. the next round's duchess_score_active, so the order per round
 * is score(k+1) -> kv_round(k) -> duchess_round(k+1). */
#define DUCHESS_KV_OVERLAP 1
/* launched right after the engine's duchess_round (waits for it), releasing
 * the next launch at once: the next round's duchess_score_active_ex with
 * DUCHESS_SCORE_NO_INPUT_WAIT streams beside this update and completes only
 * after it, so the round after that sees the KV update done. */
#define DUCHESS_KV_LEAD 2

typedef struct DuchessKV {
  int32_t block_tokens;       /* tokens per block (16) */
  int32_t blocks_per_slot;    /* P */
  int32_t max_blocks;         /* table width: blocks per branch row */
  int32_t flags;              /* DUCHESS_KV_OVERLAP or DUCHESS_KV_LEAD */
  int64_t kv_bytes_per_token; /* bytes of KV per token (one layer slice: 2*8*128*2) */
  int32_t* table;             /* [R*Bmax*max_blocks] */
  int32_t* kv_tokens;         /* [R*Bmax] tokens each row's blocks cover */
  int32_t* refcount;          /* [R*P] by global block id */
  int32_t* free_stack;        /* [R*P] local block ids */
  int32_t* arena;             /* [R*4] */
  int32_t* jobs;              /* [R*C*4] this round's tail copies (src, dst, tokens, -) */
  int32_t* job_count;         /* [R] */
  char* kv_pool;              /* [R*P*block_tokens*kv_bytes_per_token] or NULL */
  long long* counters;        /* [DUCHESS_KV_N_COUNTERS] */
} DuchessKV;

/* Apply the round just completed by duchess_round (or, before the first round,
 * the engine's first duchess_advance) to the KV cache, per slot in fixed order:
 * (1) the round's forks (DuchessState.forks, record order) whose child is still
 * active: the child row gets the root's first prefix/block_tokens blocks
 * (refcount += 1) and a fresh block with a copy of the root's partial tail
 * (prefix % block_tokens tokens of KV bytes); (2) rows of branches that are no
 * longer active release their blocks (refcount -= 1; 0 -> pushed on the free
 * stack, by branch id then block index); (3) active rows grow to
 * ceil(position / block_tokens) blocks (popped from the stack, then above the
 * high-water mark). A slot whose request finished this round resets its arena
 * first. Deterministic: a request's tables depend only on its own rounds.
 * Tail KV bytes are copied by the same launch. Must run before the next
 * duchess_round (which rewrites the round records and branch fields read). */
int duchess_kv_round(const DuchessPolicy* policy, const DuchessState* state, const DuchessKV* kv,
                     void* stream);

/* ---- K4: logistic-regression gradient for probe training ------------------
 * grad[h] = inv_n * sum_i (sigmoid(x_i . w + w[H]) - y_i) x_ih, grad[H] = the
 * bias term; w and grad are [H+1] fp32 (bias last). One HBM pass over X. */
size_t duchess_lr_grad_workspace_bytes(int32_t H);
int duchess_lr_grad(const void* X, int32_t dtype, const float* y, const float* w,
                    int64_t n_rows, int32_t H, float inv_n, float* grad_out, void* workspace,
                    size_t workspace_bytes, void* stream);
int duchess_sgd_update(float* w, const float* grad, int32_t n, float lr, void* stream);

/* Build/runtime introspection. */
/* Measurement: stream `bytes` of device memory (16-byte aligned) through a
 * read-only persistent kernel (the read-only HBM ceiling, bench.py roofline). */
int duchess_read_stream(const void* buf, int64_t bytes, uint32_t* sink, void* stream);
/* Measurement: write `bytes` of device memory (16-byte aligned) with a
 * persistent streaming-store kernel (the write-only HBM ceiling, bench.py). */
int duchess_write_stream(void* buf, int64_t bytes, uint32_t seed, void* stream);
/* Measurement: hold `stream` until the host writes nonzero to *host_flag
 * (pinned host memory) or timeout_ns elapses (then *timed_out = 1, device
 * memory), so a benchmark can enqueue its whole timed region first. */
int duchess_gate(const int32_t* host_flag, int64_t timeout_ns, int32_t* timed_out, void* stream);

const char* duchess_version(void);
int duchess_device_arch(void);

#ifdef __cplusplus
}
#endif
#endif /* DUCHESS_B200_H */
