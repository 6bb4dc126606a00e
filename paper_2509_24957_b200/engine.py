"""BatchedDuchess — the device-resident DUCHESS orchestration engine.

Holds the SoA state of R request slots (each with up to C = max_branches
branch slots) in device memory and advances all of them one round per
``step()``: ``duchess_advance`` (refill + phase 1) -> ``duchess_score`` (K1,
when predictions come from probe scores) -> ``duchess_decide`` (phases 2-5).
Requests enter slots from a service queue (FCFS or difficulty order, see
scheduler.py) and finished slots are refilled on device, so a run needs no
host synchronisation between rounds.

Per-request semantics are exactly the reference's DuchessRun
(orchestrator.py:316-402); the host only packs traces (workload.py:35-60) and
unpacks RoundReports / RequestOutcomes.
"""

from __future__ import annotations

import ctypes
import math
import random
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

NO_ANSWER = ""


def at_least(frac: float, slots: int) -> int:
    """orchestrator.py:162-164."""
    return math.ceil(frac * slots - 1e-9)


def mt_state_words(rng_or_seed) -> np.ndarray:
    """625 uint32 words (624 MT19937 words + index) of a random.Random."""
    rng = rng_or_seed if isinstance(rng_or_seed, random.Random) else random.Random(rng_or_seed)
    version, internal, _gauss = rng.getstate()
    if version != 3 or len(internal) != _lib.MT_WORDS:
        raise ValueError("unsupported random.Random state layout")
    return np.asarray(internal, dtype=np.uint32)


MT_PRISTINE = 0x80000000   # slot MT index flag: words still live in the pool's mt_init


def pretwist(words: np.ndarray) -> np.ndarray:
    """The same MT19937 stream with its pending twist done: a freshly seeded
    state (index 624) becomes the regenerated words with index 0, so the
    device draws a fresh request's first words without a twist."""
    words = np.asarray(words, dtype=np.uint32)
    if int(words[-1]) < _lib.MT_WORDS - 1:
        return words
    r = random.Random()
    r.setstate((3, tuple(int(x) for x in words), None))
    r.getrandbits(32)                       # runs the twist, consumes word 0
    out = np.asarray(r.getstate()[1], dtype=np.uint32)
    out[-1] = 0
    return out


def seed_states(seeds, out: torch.Tensor | None = None, device="cuda") -> torch.Tensor:
    """random.Random(seed).getstate() words for many int seeds, pre-twisted
    (index 0, as pretwist), built on the device by duchess_mt_seed: [n * 625]."""
    n = len(seeds)
    lib = _lib.load()
    dev = out.device if out is not None else torch.device(device)
    if out is None:
        out = torch.empty(max(n, 1) * _lib.MT_WORDS, dtype=torch.int32, device=dev)
    sd = torch.from_numpy(np.asarray([int(x) for x in seeds], dtype=np.uint64).view(np.int64)).to(dev)
    _lib.check(lib.duchess_mt_seed(sd.data_ptr(), n, out.data_ptr(), _lib.stream_handle()),
               "duchess_mt_seed")
    return out


def set_mt_state(rng: random.Random, words: np.ndarray) -> None:
    _v, _internal, gauss = rng.getstate()
    rng.setstate((3, tuple(int(x) for x in words), gauss))


@dataclass
class PackedWorkload:
    """Device tables for a pool of traces; answers interned per request."""
    answers: list            # per request: list of answer strings, id order
    n_templates: np.ndarray  # [P]
    tensors: dict
    struct: _lib.Workload
    branch_cap: int
    answer_cap: int
    tmpl_off: np.ndarray | None = None   # host copy [P + 1] (queue records)
    mt_index: np.ndarray | None = None   # host MT index word per request (None: device-seeded, 0)

    def with_queue(self, queue, cycle: bool) -> "PackedWorkload":
        """The same (shared, read-only) tables with another service queue:
        request shards of one pool (several engines on one GPU, or one rank's
        share of the workload) pack the traces once."""
        dev = self.tensors["tmpl_off"].device
        tens = dict(self.tensors)
        tens.update(_queue_tensors(queue, self.tmpl_off, self.mt_index, dev))
        st = _lib.Workload()
        st.n_requests = self.struct.n_requests
        st.queue_len = len(queue)
        st.cycle = 1 if cycle else 0
        for k, v in tens.items():
            setattr(st, k, v.data_ptr())
        return PackedWorkload(self.answers, self.n_templates, tens, st, self.branch_cap,
                              self.answer_cap, self.tmpl_off, self.mt_index)


def _queue_tensors(queue, tmpl_off, mt_index, device) -> dict:
    """Service queue + per position (pool index, template base, template
    count, MT index word) records: one 16-byte load per refill."""
    q = np.asarray(list(queue), dtype=np.int64).reshape(-1)
    out = {"queue": torch.tensor(q.astype(np.int32) if len(q) else np.zeros(1, np.int32),
                                 dtype=torch.int32, device=device)}
    if len(q):
        toff = np.asarray(tmpl_off, dtype=np.int64)
        idx = np.zeros(len(q), dtype=np.int64) if mt_index is None else mt_index[q]
        rec = np.stack([q, toff[q], toff[q + 1] - toff[q], idx.astype(np.int64)],
                       axis=1).astype(np.int32)
        out["queue_rec"] = torch.from_numpy(np.ascontiguousarray(rec).reshape(-1)).to(device)
    return out


def intern_answers(trace) -> list[str]:
    """Sorted distinct answers of a request with "" first, so answer-id order
    equals string order (majority_vote tie-break, core.py:83)."""
    s = {NO_ANSWER, trace.ground_truth}
    for t in trace.templates:
        s.add(t.final_answer)
        s.update([a for _, a in t.probes])
    return sorted(s)


def pack_workload(traces, mt_words, queue, cycle: bool, device) -> PackedWorkload:
    """Trace ingestion into the device SoA tables (workload.py:35-60): CSR
    template / probe / prediction arrays with per-request interned answers."""
    P = len(traces)
    tmpl_off = [0]
    gt, nat, fin, conv = [], [], [], []
    probe_n, probe_at, probe_ans = [], [], []
    pred_n, pred_at, pred_p = [], [], []
    answers = []
    for tr in traces:
        ans = intern_answers(tr)
        idx = {a: i for i, a in enumerate(ans)}.__getitem__
        answers.append(ans)
        gt.append(idx(tr.ground_truth))
        tm = tr.templates
        nat += [t.natural_length for t in tm]
        fin += [idx(t.final_answer) for t in tm]
        conv += [-1 if t.oracle_convergence is None else t.oracle_convergence for t in tm]
        for t in tm:
            pr = t.probes
            probe_n.append(len(pr))
            probe_at += [at for at, _ in pr]
            probe_ans += [idx(a) for _, a in pr]
            pp = t.pred_probs or ()
            pred_n.append(len(pp))
            if pp:
                pred_at += [at for at, _ in pp]
                pred_p += [float(p) for _, p in pp]
        tmpl_off.append(len(nat))
    probe_off = np.concatenate([[0], np.cumsum(probe_n, dtype=np.int64)]) if probe_n else [0]
    pred_off = np.concatenate([[0], np.cumsum(pred_n, dtype=np.int64)]) if pred_n else [0]

    def i32(x):
        return torch.tensor(np.asarray(x, dtype=np.int32).reshape(-1) if len(x) else
                            np.zeros(1, np.int32), dtype=torch.int32, device=device)

    tens = {
        "tmpl_off": i32(tmpl_off), "ground_truth": i32(gt), "nat_len": i32(nat),
        "final_ans": i32(fin), "conv": i32(conv), "probe_off": i32(probe_off),
        "probe_at": i32(probe_at), "probe_ans": i32(probe_ans), "pred_off": i32(pred_off),
        "pred_at": i32(pred_at),
        "pred_p": torch.tensor(np.asarray(pred_p if pred_p else [0.0], dtype=np.float64),
                               device=device),
        "mt_init": (torch.empty(max(P, 1) * _lib.MT_WORDS, dtype=torch.int32, device=device)
                    if mt_words is None else
                    torch.from_numpy(np.ascontiguousarray(mt_words, dtype=np.uint32).view(np.int32))
                    .reshape(-1).to(device)),
    }
    # device-seeded states are pre-twisted: index 0
    mt_index = (None if mt_words is None else
                np.ascontiguousarray(mt_words, dtype=np.uint32).reshape(-1, _lib.MT_WORDS)[:, -1]
                .astype(np.int64))
    toff_h = np.asarray(tmpl_off, dtype=np.int64)
    tens.update(_queue_tensors(queue, toff_h, mt_index, device))
    st = _lib.Workload()
    st.n_requests = P
    st.queue_len = len(queue)
    st.cycle = 1 if cycle else 0
    for k, v in tens.items():
        setattr(st, k, v.data_ptr())
    n_t = np.diff(np.asarray(tmpl_off))
    return PackedWorkload(answers, n_t, tens, st, int(max(n_t.max() if P else 1, 1)),
                          int(max(len(a) for a in answers) if P else 1), toff_h, mt_index)


def pack_pool(traces, seeds, device, queue=None, cycle: bool = False) -> PackedWorkload:
    """Pack a pool of traces with their per-request RNG streams: int seeds are
    expanded to random.Random(seed) states on the device (duchess_mt_seed),
    random.Random objects are copied from the host."""
    P = len(traces)
    queue = list(range(P)) if queue is None else list(queue)
    int_seeds = P > 0 and all(isinstance(s, (int, np.integer)) and not isinstance(s, bool)
                              and 0 <= int(s) < (1 << 64) for s in seeds)
    if int_seeds:
        mt = None
    else:
        mt = (np.stack([pretwist(mt_state_words(s)) for s in seeds]) if P
              else np.zeros((0, 625), np.uint32))
    wl = pack_workload(traces, mt, queue, cycle, device)
    if int_seeds:
        seed_states(seeds, wl.tensors["mt_init"])
    return wl


_KINDS = {_lib.ACT_CONTINUE: "continue", _lib.ACT_TERMINATE: "terminate",
          _lib.ACT_BRANCH_OUT: "branch_out"}


def decode_round(round_rec: np.ndarray, actions: np.ndarray, R: int, C: int):
    """(pool index, RoundReport-tuple) per slot that ran a round, from host
    copies of DuchessState.round_rec [R*REC_WORDS] and actions [R*2C*3]."""
    rec = np.asarray(round_rec).reshape(R, _lib.REC_WORDS)
    acts = np.asarray(actions).reshape(R, 2 * C, 3)
    out = []
    for r in np.nonzero(rec[:, _lib.REC_ROUND])[0]:
        rr = rec[r]
        n = int(rr[_lib.REC_NACTIONS])
        actions_r = [(_KINDS[int(a[0])], int(a[1]), None if a[2] < 0 else int(a[2]))
                     for a in acts[r, :n]]
        out.append((int(rr[_lib.REC_REQ]),
                    (int(rr[_lib.REC_ROUND]), int(rr[_lib.REC_DECODING]),
                     int(rr[_lib.REC_MAX_CHUNK]), int(rr[_lib.REC_DECODE]),
                     int(rr[_lib.REC_PROBES]), actions_r, bool(rr[_lib.REC_DONE]))))
    return out


class BatchedDuchess:
    """R request slots advanced in lockstep rounds on one GPU.

    traces:   list of RequestTrace-like objects (templates, ground_truth).
    config:   OrchestratorConfig-like (max_branches, interval_tokens, ...).
    seeds:    per-request int seeds or random.Random objects (DuchessRun's rng).
    pred_source: _lib.PRED_TRACE (reference default predictor: pred_probs, else
              synthetic with rho), _lib.PRED_DEVICE (K1 probe scores) or
              _lib.PRED_HOST (caller-provided probabilities by slot).
    """

    def __init__(self, traces, config, seeds, n_slots: int | None = None, *,
                 pred_source: int = _lib.PRED_TRACE, rho: float = 1.0, queue=None,
                 cycle: bool = False, n_layers: int = 1, combine: int = 0,
                 policy: str = "duchess", device: str | torch.device = "cuda",
                 packed: PackedWorkload | None = None):
        _lib.require_cuda()
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.traces = traces
        self.config = config
        c = int(config.max_branches)
        if not 1 <= c <= _lib.MAX_SLOTS:
            raise ValueError(f"max_branches must be in [1, {_lib.MAX_SLOTS}] on device")
        P = len(traces)
        self.P, self.C = P, c
        self.R = n_slots if n_slots is not None else P
        queue = list(range(P)) if queue is None else list(queue)
        if packed is not None:         # shared tables of one pool (pack_pool), own queue
            if packed.struct.n_requests != P:
                raise ValueError("packed workload does not match the traces")
            self.wl = packed.with_queue(queue, cycle)
        else:
            self.wl = pack_pool(traces, seeds, self.device, queue=queue, cycle=cycle)
        pol = _lib.Policy()
        pol.max_branches = c
        pol.interval_tokens = int(config.interval_tokens)
        pol.early_term_rounds = int(config.early_term_rounds)
        pol.token_cap = int(config.token_cap)
        pol.probe_cost_tokens = int(config.probe_cost_tokens)
        pol.need_consensus = at_least(config.consensus_frac, c)
        pol.need_coverage = at_least(config.coverage_frac, c)
        pol.pred_source = int(pred_source)
        pol.n_layers = int(n_layers)
        pol.combine = int(combine)
        pol.early_term_threshold = float(config.early_term_threshold)
        pol.inv_temperature = 1.0 / config.branch_out_temperature     # orchestrator.py:182
        pol.rho = float(rho)
        kinds = {"duchess": _lib.POLICY_DUCHESS, "default-sc": _lib.POLICY_DEFAULT_SC,
                 "short-mk": _lib.POLICY_SHORT_MK, "dynasor": _lib.POLICY_DYNASOR}
        if policy not in kinds:
            raise ValueError(f"unknown policy {policy!r}")
        pol.policy_kind = kinds[policy]
        pol.short_m = int(getattr(config, "short_m", 5))
        pol.dynasor_window = int(getattr(config, "dynasor_window", 3))
        self.policy_name = policy
        self.policy = pol
        self._alloc_state()

    # ------------------------------------------------------------------
    def _alloc_state(self) -> None:
        R, C, dev = self.R, self.C, self.device
        B, A = self.wl.branch_cap, self.wl.answer_cap
        i32 = dict(dtype=torch.int32, device=dev)
        t = {}
        for name in ("slot_req", "n_branches", "next_template", "tokens_decode",
                     "tokens_probe", "rounds"):
            t[name] = torch.zeros(R, **i32)
        t["slot_req"].fill_(-1)
        t["needs_refill"] = torch.ones(R, **i32)
        t["done"] = torch.ones(R, **i32)
        t["tally"] = torch.zeros(R * A, **i32)
        t["mt"] = torch.zeros(R * _lib.MT_WORDS, **i32)
        for name in ("br_offset", "br_decoded", "br_streak", "br_status", "br_final",
                     "br_npred", "br_slot"):
            t[name] = torch.zeros(R * B, **i32)
        t["br_last_pred"] = torch.zeros(R * B, dtype=torch.float64, device=dev)
        t["br_probe_last"] = torch.full((R * B,), -1, **i32)
        t["br_probe_run"] = torch.zeros(R * B, **i32)
        t["slot_aux"] = torch.zeros(R, **i32)
        t["slot_branch"] = torch.full((R * C,), -1, **i32)
        t["row_mask"] = torch.zeros(R * C, dtype=torch.uint8, device=dev)
        t["row_pos"] = torch.zeros(R * C, **i32)
        t["row_tmpl"] = torch.zeros(R * C, **i32)
        t["row_req"] = torch.zeros(R * C, dtype=torch.int64, device=dev)
        t["p1_rec"] = torch.zeros(R * 8, **i32)
        t["round_rec"] = torch.zeros(R * _lib.REC_WORDS, **i32)
        t["actions"] = torch.zeros(R * 2 * C * 3, **i32)
        t["forks"] = torch.zeros(R * C * 4, **i32)
        t["step_pred"] = torch.zeros(R * C, dtype=torch.float64, device=dev)
        t["queue_head"] = torch.zeros(2, **i32)
        t["active_rows"] = torch.zeros(2 * R * C, **i32)
        t["active_count"] = torch.zeros(8, **i32)       # see DuchessState.active_count
        P = max(self.P, 1)
        for name in ("out_final", "out_reason", "out_tokens_decode", "out_tokens_probe",
                     "out_rounds", "out_error"):
            t[name] = torch.full((P,), -1, **i32)
        t["out_tally"] = torch.zeros(P * A, **i32)
        t["counters"] = torch.zeros(_lib.N_COUNTERS, dtype=torch.int64, device=dev)
        self.t = t
        st = _lib.State()
        st.n_slots, st.branch_cap, st.answer_cap = R, B, A
        for name in _lib.STATE_PTR_FIELDS:
            if name in t:
                setattr(st, name, t[name].data_ptr())
        self.state = st
        self.probs = torch.zeros(R * C * max(self.policy.n_layers, 1), dtype=torch.float64,
                                 device=dev)

    # ------------------------------------------------------------------
    def enable_trace(self) -> torch.Tensor:
        """Per-slot decide phase timestamps (globaltimer ns) for profiling."""
        self.t["trace"] = torch.zeros(self.R * _lib.TRACE_WORDS, dtype=torch.int64,
                                      device=self.device)
        self.state.trace = self.t["trace"].data_ptr()
        return self.t["trace"]

    def advance(self, stream=None) -> None:
        """Refill finished slots, then phase 1 (orchestrator.py:344-355)."""
        _lib.check(self.lib.duchess_advance(self.policy, self.wl.struct, self.state,
                                            _lib.stream_handle(stream)), "duchess_advance")

    def decide(self, probs: torch.Tensor | None = None, stream=None) -> None:
        """Phases 2-5 (orchestrator.py:357-402). probs: [R*C*L] fp64 by slot,
        required for PRED_DEVICE / PRED_HOST."""
        p = probs if probs is not None else self.probs
        _lib.check(self.lib.duchess_decide(self.policy, self.wl.struct, self.state,
                                           p.data_ptr(), _lib.stream_handle(stream)),
                   "duchess_decide")

    def round(self, probs: torch.Tensor | None = None, stream=None) -> None:
        """Fused decide(k) + advance(k+1) (duchess_round, one launch, no grid
        barrier). After it, round_reports() describe round k and the row mask /
        active list describe the survivors of round k+1."""
        p = probs if probs is not None else self.probs
        _lib.check(self.lib.duchess_round(self.policy, self.wl.struct, self.state,
                                          p.data_ptr(), _lib.stream_handle(stream)),
                   "duchess_round")

    def upload_survivors(self, host_acts: torch.Tensor, dev_acts: torch.Tensor,
                         stream=None) -> None:
        """Copy only the survivor rows of the round in flight (the active list)
        from pinned host memory host_acts [R*C, ...] into the same rows of
        dev_acts (duchess_gather_active: one kernel, PCIe reads of the listed
        rows only). Both arrays contiguous with identical shape / dtype."""
        if host_acts.shape != dev_acts.shape or host_acts.dtype != dev_acts.dtype:
            raise ValueError("host and device activation arrays must match")
        if not host_acts.is_pinned() or not dev_acts.is_cuda:
            raise ValueError("host_acts must be pinned host memory, dev_acts a CUDA tensor")
        if not (host_acts.is_contiguous() and dev_acts.is_contiguous()):
            raise ValueError("activation arrays must be contiguous")
        rows = host_acts.shape[0]
        if rows != self.R * self.C:
            raise ValueError("activation arrays must have R*C rows")
        row_bytes = host_acts[0].numel() * host_acts.element_size()
        _lib.check(self.lib.duchess_gather_active(
            host_acts.data_ptr(), dev_acts.data_ptr(), row_bytes,
            self.t["active_rows"].data_ptr(), self.t["active_count"].data_ptr(), rows,
            _lib.stream_handle(stream)), "duchess_gather_active")

    def survivor_rows_host(self, stream=None) -> np.ndarray:
        """The survivor rows the next scorer launch reads, read back to the
        host (waits for the stream: the round that listed them must be done)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream()
        st.synchronize()
        cnt = self.t["active_count"].cpu().numpy()
        par = int(cnt[2])
        n = int(cnt[par])
        rows = self.R * self.C
        return self.t["active_rows"][par * rows: par * rows + n].cpu().numpy()

    def upload_rows(self, host_acts: torch.Tensor, dev_acts: torch.Tensor, rows,
                    stream=None) -> None:
        """DMA flavour of upload_survivors for a survivor list the caller holds
        on the host (e.g. survivor_rows_host()): runs of consecutive rows, one
        cudaMemcpyAsync each (duchess_upload_rows)."""
        if host_acts.shape != dev_acts.shape or host_acts.dtype != dev_acts.dtype:
            raise ValueError("host and device activation arrays must match")
        if not host_acts.is_pinned() or not dev_acts.is_cuda:
            raise ValueError("host_acts must be pinned host memory, dev_acts a CUDA tensor")
        if not (host_acts.is_contiguous() and dev_acts.is_contiguous()):
            raise ValueError("activation arrays must be contiguous")
        r = np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
        row_bytes = host_acts[0].numel() * host_acts.element_size()
        _lib.check(self.lib.duchess_upload_rows(
            host_acts.data_ptr(), dev_acts.data_ptr(), row_bytes,
            r.ctypes.data_as(ctypes.c_void_p), len(r), host_acts.shape[0],
            _lib.stream_handle(stream)), "duchess_upload_rows")

    def active_list(self):
        """(rows, count) device views of the survivor list the next scorer
        launch reads (duchess_score_list): the parity duchess_round flips
        lives on the device, so the views are chosen on the device too."""
        return self.t["active_rows"], self.t["active_count"]

    def baseline_round(self, stream=None) -> None:
        """One round of a baseline policy (Default SC / Short-m@k / Dynasor)."""
        _lib.check(self.lib.duchess_baseline_round(self.policy, self.wl.struct, self.state,
                                                   _lib.stream_handle(stream)),
                   "duchess_baseline_round")

    def step(self, score_fn=None, stream=None) -> None:
        """One round for every occupied slot. score_fn(engine) must fill
        self.probs for the survivors flagged in t['row_mask'] when the
        prediction source is PRED_DEVICE (e.g. fill + K1)."""
        if self.policy.policy_kind != _lib.POLICY_DUCHESS:
            self.baseline_round(stream)
            return
        self.advance(stream)
        if self.policy.pred_source != _lib.PRED_TRACE:
            if score_fn is None:
                raise ValueError("this prediction source needs a score_fn")
            score_fn(self)
        self.decide(stream=stream)

    # ------------------------------------------------------------------
    def counters(self) -> np.ndarray:
        return self.t["counters"].cpu().numpy()

    def all_done(self) -> bool:
        done = self.t["done"].cpu().numpy()
        head = int(self.t["queue_head"][0])
        return bool(done.all()) and head >= self.wl.struct.queue_len

    def round_reports(self):
        """Per-slot (pool index, RoundReport-tuple) of the latest round:
        (round_index, decoding, max_chunk, decode_tokens, probes,
        [(kind, branch_id, source_or_None)], done)."""
        return decode_round(self.t["round_rec"].cpu().numpy(), self.t["actions"].cpu().numpy(),
                            self.R, self.C)

    def outcomes(self):
        """Per pool index: None (unfinished) or dict(tally, final, reason,
        tokens_decode, tokens_probe, rounds, error)."""
        t = {k: self.t[k].cpu().numpy() for k in
             ("out_final", "out_reason", "out_tokens_decode", "out_tokens_probe",
              "out_rounds", "out_error")}
        tally = self.t["out_tally"].view(max(self.P, 1), self.wl.answer_cap).cpu().numpy()
        reasons = {1: "consensus", 2: "coverage", 3: "exhausted"}
        res = []
        for p in range(self.P):
            if t["out_reason"][p] < 0:
                res.append(None)
                continue
            ans = self.wl.answers[p]
            counts = {ans[a]: int(n) for a, n in enumerate(tally[p][:len(ans)]) if n}
            fin = int(t["out_final"][p])
            res.append(dict(tally=counts, final=None if fin < 0 else ans[fin],
                            reason=reasons[int(t["out_reason"][p])],
                            tokens_decode=int(t["out_tokens_decode"][p]),
                            tokens_probe=int(t["out_tokens_probe"][p]),
                            rounds=int(t["out_rounds"][p]), error=int(t["out_error"][p])))
        return res

    def slot_mt_state(self, slot: int) -> np.ndarray:
        """625-word MT19937 state (words + index) of a slot's request,
        resolving the copy-on-write pool state (MT_PRISTINE)."""
        W = _lib.MT_WORDS
        st = self.t["mt"][slot * W:(slot + 1) * W].cpu().numpy().view(np.uint32).copy()
        if int(st[-1]) & MT_PRISTINE:
            p = int(self.t["slot_req"][slot])
            init = self.wl.tensors["mt_init"][p * W:(p + 1) * W].cpu().numpy().view(np.uint32)
            st[:-1] = init[:-1]
            st[-1] = int(st[-1]) & ~MT_PRISTINE
        return st

    def branch_snapshot(self, slot: int):
        """Host copy of one slot's branch table (for facades / tests)."""
        B = self.wl.branch_cap
        sl = slice(slot * B, (slot + 1) * B)
        g = {k: self.t[k][sl].cpu().numpy() for k in
             ("br_offset", "br_decoded", "br_streak", "br_status", "br_final", "br_npred",
              "br_last_pred", "br_slot")}
        n = int(self.t["n_branches"][slot])
        return {k: v[:n] for k, v in g.items()}
