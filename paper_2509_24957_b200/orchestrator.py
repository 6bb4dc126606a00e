"""Per-request policy API (mirrors reference orchestrator.py), GPU-backed.

``DuchessRun(trace, config, rng, synthetic=None, predictor=None)`` keeps the
reference signature and semantics; each ``step()`` runs one round of the
device engine (engine.BatchedDuchess, one slot) — ``duchess_advance`` then
``duchess_decide`` — and mirrors the device state back into reference-shaped
``BranchState`` / ``RoundReport`` / ``RequestOutcome`` objects. The caller's
``rng`` is advanced exactly as the reference advances it (device MT19937
state is synchronised both ways every step).

Prediction sources (orchestrator.py:211-224, :319-327):
* ``predictor=None`` or ``make_correctness_predictor(...)``: trace-embedded
  pred_probs else the synthetic oracle, evaluated on the device;
* any other callable: invoked on the host per surviving branch in creation
  order (the reference seam), its probabilities uploaded for the decision.
For throughput use engine.BatchedDuchess directly (many requests per launch,
probabilities from the K1 scorer).

The rule primitives (branch_out_weights / branch_out_sample,
check_request_termination, check_early_termination) are the same device
functions K2 uses, exposed one call at a time.
"""

from __future__ import annotations

import logging
import math
import random
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import VoteTally
from .predictor import SyntheticPredictorConfig
from .workload import BranchTemplate, RequestTrace

logger = logging.getLogger(__name__)

ACTIVE = "active"
EARLY_TERMINATED = "early_terminated"
NATURAL_END = "natural_end"
CAPPED = "capped"
CANCELLED = "cancelled"
CONSENSUS = "consensus"
COVERAGE = "coverage"
EXHAUSTED = "exhausted"
POLICY_DUCHESS = "duchess"
POLICY_DEFAULT_SC = "default-sc"
POLICY_SHORT_MK = "short-mk"
POLICY_DYNASOR = "dynasor"
POLICIES = (POLICY_DUCHESS, POLICY_DEFAULT_SC, POLICY_SHORT_MK, POLICY_DYNASOR)
BRANCH_PROB_FLOOR = 1e-6
TERMINATION_DISABLED = math.inf

_STATUS = {_lib.ACTIVE: ACTIVE, _lib.EARLY_TERMINATED: EARLY_TERMINATED,
           _lib.NATURAL_END: NATURAL_END, _lib.CAPPED: CAPPED, _lib.CANCELLED: CANCELLED}
_REASON = {_lib.REASON_CONSENSUS: CONSENSUS, _lib.REASON_COVERAGE: COVERAGE,
           _lib.REASON_EXHAUSTED: EXHAUSTED}


@dataclass(frozen=True)
class OrchestratorConfig:
    """All intra-request policy knobs (orchestrator.py:62-96)."""
    max_branches: int = 10
    interval_tokens: int = 16
    early_term_threshold: float = 0.7
    early_term_rounds: int = 2
    branch_out_temperature: float = 1.0
    consensus_frac: float = 0.6
    coverage_frac: float = 0.8
    token_cap: int = 4096
    probe_cost_tokens: int = 10
    dynasor_window: int = 3
    short_m: int = 5

    def __post_init__(self) -> None:
        checks = (
            (self.max_branches >= 1, "max_branches must be >= 1"),
            (self.interval_tokens >= 1, "interval_tokens must be >= 1"),
            (self.early_term_rounds >= 1, "early_term_rounds must be >= 1"),
            (self.branch_out_temperature > 0, "branch_out_temperature must be > 0"),
            (0.0 < self.consensus_frac <= 1.0, "consensus_frac must be in (0, 1]"),
            (self.consensus_frac <= self.coverage_frac <= 1.0,
             "coverage_frac must be in [consensus_frac, 1]"),
            (self.token_cap >= self.interval_tokens, "token_cap must be >= interval_tokens"),
            (self.probe_cost_tokens >= 0, "probe_cost_tokens must be >= 0"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


@dataclass
class BranchState:
    branch_id: int
    template_index: int
    template: BranchTemplate
    offset_base: int = 0
    tokens_decoded: int = 0
    prediction_history: list = field(default_factory=list)
    probe_history: list = field(default_factory=list)
    streak: int = 0
    status: str = ACTIVE
    final_answer: str | None = None
    last_prediction: float = 0.5

    @property
    def position(self) -> int:
        return self.offset_base + self.tokens_decoded


@dataclass(frozen=True)
class BranchAction:
    kind: str
    branch_id: int
    source_branch_id: int | None = None


@dataclass
class RequestOutcome:
    tally: VoteTally
    final: str
    termination_reason: str
    tokens_decode: int
    tokens_probe: int
    rounds: int

    @property
    def tokens_total(self) -> int:
        return self.tokens_decode + self.tokens_probe


@dataclass
class RoundReport:
    round_index: int
    decoding_branches: int
    max_chunk: int
    decode_tokens: int
    probes: int
    actions: list
    done: bool


def _at_least(frac: float, slots: int) -> int:
    return math.ceil(frac * slots - 1e-9)


# ---------------------------------------------------------------------------
# rule primitives, on the device

def check_early_termination(branch: BranchState, threshold: float, rounds: int) -> bool:
    """Last ``rounds`` predictions all strictly above threshold (:167-174)."""
    import torch
    _lib.require_cuda()
    lib = _lib.load()
    h = torch.tensor(list(branch.prediction_history) or [0.0], dtype=torch.float64,
                     device="cuda")
    off = torch.tensor([0, len(branch.prediction_history)], dtype=torch.int32, device="cuda")
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.duchess_early_termination(h.data_ptr(), off.data_ptr(), 1, float(threshold),
                                             int(rounds), out.data_ptr(), _lib.stream_handle()),
               "duchess_early_termination")
    return bool(int(out))


def _branch_out(probs, temperature: float, rng: random.Random | None, n_draws: int):
    import torch

    from .engine import mt_state_words, set_mt_state
    if len(probs) == 0:
        raise ValueError("no branch to duplicate")
    _lib.require_cuda()
    lib = _lib.load()
    p = torch.tensor([float(x) for x in probs], dtype=torch.float64, device="cuda")
    w = torch.empty_like(p)
    idx = torch.empty(max(n_draws, 1), dtype=torch.int32, device="cuda")
    st = None
    if n_draws:
        st = torch.from_numpy(mt_state_words(rng).view(np.int32).copy()).cuda()
    amb = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(lib.duchess_branch_out_sample(p.data_ptr(), len(probs), 1.0 / temperature,
                                             _lib.ptr(st), n_draws, idx.data_ptr(),
                                             w.data_ptr(), amb.data_ptr(),
                                             _lib.stream_handle()), "duchess_branch_out_sample")
    if st is not None:
        set_mt_state(rng, st.cpu().numpy().view(np.uint32))
    return [float(x) for x in w.cpu().numpy()], [int(i) for i in idx.cpu().numpy()[:n_draws]]


def branch_out_weights(probs, temperature: float) -> list:
    """p^(1/temperature) renormalised (:177-185)."""
    return _branch_out(probs, temperature, None, 0)[0]


def branch_out_sample(probs, temperature: float, rng: random.Random) -> int:
    """One draw from the rescaled distribution (:188-197)."""
    return _branch_out(probs, temperature, rng, 1)[1][0]


def branch_out_sample_many(probs, temperature: float, rng: random.Random, n: int) -> list:
    """n sequential branch_out_sample calls sharing one rng, one launch."""
    return _branch_out(probs, temperature, rng, n)[1]


def check_request_termination(tally: VoteTally, consensus_frac: float, coverage_frac: float,
                              max_branches: int) -> str | None:
    """Consensus first, then coverage (:200-208)."""
    from .core import _device_vote
    answers = sorted(tally.counts)
    _, why = _device_vote([tally.counts[a] for a in answers],
                          _at_least(consensus_frac, max_branches),
                          _at_least(coverage_frac, max_branches))
    return _REASON.get(why)


# ---------------------------------------------------------------------------
# predictor seam

class _DefaultPredictor:
    """make_correctness_predictor: pred_probs if present else the synthetic
    oracle. Recognised by DuchessRun and evaluated on the device."""

    def __init__(self, trace: RequestTrace, synthetic: SyntheticPredictorConfig):
        self.trace, self.synthetic = trace, synthetic

    def __call__(self, template, position, rng):
        from .predictor import synthetic_predict
        from .workload import probe_answer, trace_prediction
        if template.pred_probs:
            return trace_prediction(template, position)
        return synthetic_predict(probe_answer(template, position) == self.trace.ground_truth,
                                 self.synthetic, rng)


def make_correctness_predictor(trace: RequestTrace, synthetic: SyntheticPredictorConfig):
    return _DefaultPredictor(trace, synthetic)


# ---------------------------------------------------------------------------
# request state machines

class RequestRun:
    """Base round-granularity state machine (orchestrator.py:227-313)."""

    def __init__(self, trace: RequestTrace, config: OrchestratorConfig,
                 rng: random.Random | None = None) -> None:
        self.trace = trace
        self.config = config
        self.rng = rng
        self.tally = VoteTally()
        self.branches: list = []
        self.tokens_decode = 0
        self.tokens_probe = 0
        self.rounds = 0
        self.outcome: RequestOutcome | None = None
        self._next_template = 0
        seeded = min(config.max_branches, len(trace.templates))
        if seeded < config.max_branches:
            logger.warning("request %s: only %d templates for %d branch slots, "
                           "parallelism degraded", trace.id, len(trace.templates),
                           config.max_branches)
        for _ in range(seeded):
            self._mirror_spawn(0, None)

    @property
    def done(self) -> bool:
        return self.outcome is not None

    def _mirror_spawn(self, offset_base: int, source) -> BranchState:
        t = self.trace.templates[self._next_template]
        b = BranchState(branch_id=len(self.branches), template_index=self._next_template,
                        template=t, offset_base=min(offset_base, t.natural_length),
                        last_prediction=source.last_prediction if source else 0.5)
        self._next_template += 1
        self.branches.append(b)
        return b

    def step(self) -> RoundReport:
        raise NotImplementedError

    def run(self) -> RequestOutcome:
        while not self.done:
            self.step()
        assert self.outcome is not None
        return self.outcome


class DuchessRun(RequestRun):
    """Prediction-guided orchestration (orchestrator.py:316-402) on the GPU."""

    def __init__(self, trace: RequestTrace, config: OrchestratorConfig, rng: random.Random,
                 synthetic: SyntheticPredictorConfig | None = None, predictor=None) -> None:
        super().__init__(trace, config, rng)
        if predictor is None:
            predictor = make_correctness_predictor(trace, synthetic or SyntheticPredictorConfig())
        self._predict = predictor
        from .engine import BatchedDuchess
        device_pred = isinstance(predictor, _DefaultPredictor) and predictor.trace is trace
        rho = predictor.synthetic.rho if device_pred else 1.0
        self._host_predictor = None if device_pred else predictor
        self._engine = BatchedDuchess(
            [trace], config, [rng if rng is not None else random.Random(0)], n_slots=1,
            pred_source=_lib.PRED_TRACE if device_pred else _lib.PRED_HOST, rho=rho)

    def _sync_rng_to_device(self) -> None:
        import torch

        from .engine import mt_state_words, pretwist
        if self.rng is None:
            return
        words = mt_state_words(self.rng)
        if self.rounds == 0:      # the refill reads the pool state (pre-twisted)
            w = torch.from_numpy(pretwist(words).view(np.int32).copy())
            tens = self._engine.wl.tensors
            tens["mt_init"].copy_(w.to(self._engine.device))
            if "queue_rec" in tens:   # the queue record caches the state's index word
                tens["queue_rec"][3] = int(w[-1])
        else:
            self._engine.t["mt"].copy_(torch.from_numpy(words.view(np.int32).copy()))

    def _sync_rng_from_device(self) -> None:
        from .engine import set_mt_state
        if self.rng is None:
            return
        st = self._engine.slot_mt_state(0)
        # index 0 only occurs in the pre-twisted initial state: nothing was
        # drawn, and the caller's rng already holds the equivalent state
        if int(st[-1]) != 0:
            set_mt_state(self.rng, st)

    def step(self) -> RoundReport:
        if self.done:
            raise RuntimeError("request already terminated")
        if self.rng is None:
            raise AssertionError("the duchess policy needs an rng")
        eng = self._engine
        self._sync_rng_to_device()
        eng.advance()
        if self._host_predictor is not None:
            self._host_predictions()
        eng.decide()
        self._sync_rng_from_device()
        return self._mirror_round()

    def _host_predictions(self) -> None:
        """The reference seam: predictor(template, position, rng) per survivor
        in creation order (:358-360); probabilities uploaded by slot."""
        import torch
        eng = self._engine
        from .engine import mt_state_words
        self._sync_rng_from_device()
        mask = eng.t["row_mask"].cpu().numpy()
        tmpl = eng.t["row_tmpl"].cpu().numpy()
        pos = eng.t["row_pos"].cpu().numpy()
        probs = np.zeros(eng.probs.numel())
        for slot in sorted(np.nonzero(mask)[0], key=lambda s: tmpl[s]):
            p = self._host_predictor(self.trace.templates[int(tmpl[slot])], int(pos[slot]),
                                     self.rng)
            probs[slot] = float(p)
        eng.probs.copy_(torch.from_numpy(probs))
        eng.t["mt"].copy_(torch.from_numpy(mt_state_words(self.rng).view(np.int32).copy()))

    def _mirror_round(self) -> RoundReport:
        eng = self._engine
        rec = eng.t["round_rec"].cpu().numpy()
        snap = eng.branch_snapshot(0)
        answers = eng.wl.answers[0]
        n_act = int(rec[_lib.REC_NACTIONS])
        acts = eng.t["actions"].view(-1, 3).cpu().numpy()[:n_act]
        kinds = {_lib.ACT_CONTINUE: "continue", _lib.ACT_TERMINATE: "terminate",
                 _lib.ACT_BRANCH_OUT: "branch_out"}
        actions = [BranchAction(kinds[int(k)], int(b), None if s < 0 else int(s))
                   for k, b, s in acts]
        for a in actions:
            if a.kind == "branch_out":
                self._mirror_spawn(int(snap["br_offset"][a.branch_id]),
                                   self.branches[a.source_branch_id])
        for b, br in enumerate(self.branches):
            old_status = br.status
            br.offset_base = int(snap["br_offset"][b])
            br.tokens_decoded = int(snap["br_decoded"][b])
            br.streak = int(snap["br_streak"][b])
            br.status = _STATUS[int(snap["br_status"][b])]
            f = int(snap["br_final"][b])
            br.final_answer = answers[f] if f >= 0 else None
            npred = int(snap["br_npred"][b])
            lp = float(snap["br_last_pred"][b])
            if npred > len(br.prediction_history):
                br.prediction_history.append(lp)
            br.last_prediction = lp
            if old_status == ACTIVE and br.status in (CAPPED, EARLY_TERMINATED):
                br.probe_history.append((br.position, br.final_answer))
        self._next_template = int(eng.t["next_template"][0])
        self.tokens_decode = int(eng.t["tokens_decode"][0])
        self.tokens_probe = int(eng.t["tokens_probe"][0])
        self.rounds = int(eng.t["rounds"][0])
        tally = eng.t["tally"].cpu().numpy()
        self.tally.counts.clear()
        for a, n in enumerate(tally[:len(answers)]):
            if n:
                self.tally.counts[answers[a]] = int(n)
        done = bool(rec[_lib.REC_DONE])
        if done:
            reason = _REASON[int(rec[_lib.REC_REASON])]
            if int(rec[_lib.REC_FINAL]) < 0:
                raise ValueError("no answers collected")
            self.outcome = RequestOutcome(self.tally, answers[int(rec[_lib.REC_FINAL])], reason,
                                          self.tokens_decode, self.tokens_probe, self.rounds)
        return RoundReport(int(rec[_lib.REC_ROUND]), int(rec[_lib.REC_DECODING]),
                           int(rec[_lib.REC_MAX_CHUNK]), int(rec[_lib.REC_DECODE]),
                           int(rec[_lib.REC_PROBES]), actions, done)


class _BaselineRun(RequestRun):
    """Device-backed baseline policy (orchestrator.py:405-561): one
    duchess_baseline_round per step, state mirrored like DuchessRun."""
    _policy = ""

    def __init__(self, trace: RequestTrace, config: OrchestratorConfig,
                 rng: random.Random | None = None) -> None:
        super().__init__(trace, config, rng)
        from .engine import BatchedDuchess
        self._engine = BatchedDuchess([trace], config, [random.Random(0)], n_slots=1,
                                      policy=self._policy)

    def step(self) -> RoundReport:
        if self.done:
            raise RuntimeError("request already terminated")
        self._engine.baseline_round()
        return DuchessRun._mirror_round(self)


class DefaultScRun(_BaselineRun):
    """Plain self-consistency (orchestrator.py:405-435)."""
    _policy = POLICY_DEFAULT_SC


class ShortMkRun(_BaselineRun):
    """Stop at the m-th finisher (orchestrator.py:438-516)."""
    _policy = POLICY_SHORT_MK

    def __init__(self, trace: RequestTrace, config: OrchestratorConfig,
                 rng: random.Random | None = None) -> None:
        if config.short_m > config.max_branches:
            raise ValueError(f"short_m ({config.short_m}) must not exceed max_branches "
                             f"({config.max_branches})")
        super().__init__(trace, config, rng)


class DynasorRun(_BaselineRun):
    """Probe every round; stop a branch on D identical answers (orchestrator.py:519-561)."""
    _policy = POLICY_DYNASOR

    def __init__(self, trace: RequestTrace, config: OrchestratorConfig,
                 rng: random.Random | None = None) -> None:
        if config.dynasor_window < 2:
            raise ValueError("dynasor_window must be >= 2")
        super().__init__(trace, config, rng)

    def step(self) -> RoundReport:
        """Every branch active at the round start and not at its natural end is
        probed this round (orchestrator.py:539-556): its probe_history gets the
        (position, answer) of every round, not only the terminal one."""
        if self.done:
            raise RuntimeError("request already terminated")
        from .workload import probe_answer
        was_active = [b.status == ACTIVE for b in self.branches]
        self._engine.baseline_round()
        kept = [len(b.probe_history) for b in self.branches]
        rep = DuchessRun._mirror_round(self)
        for b, br in enumerate(self.branches[:len(was_active)]):
            if was_active[b] and br.status != NATURAL_END:
                del br.probe_history[kept[b]:]
                br.probe_history.append((br.position, probe_answer(br.template, br.position)))
        return rep


def make_request_run(policy: str, trace: RequestTrace, config: OrchestratorConfig,
                     rng: random.Random | None = None,
                     synthetic: SyntheticPredictorConfig | None = None) -> RequestRun:
    if policy == POLICY_DUCHESS:
        if rng is None:
            raise ValueError("the duchess policy needs an rng")
        return DuchessRun(trace, config, rng, synthetic=synthetic)
    if policy == POLICY_DEFAULT_SC:
        return DefaultScRun(trace, config)
    if policy == POLICY_SHORT_MK:
        return ShortMkRun(trace, config)
    if policy == POLICY_DYNASOR:
        return DynasorRun(trace, config)
    raise ValueError(f"unknown policy {policy!r}")


def run_duchess(trace: RequestTrace, config: OrchestratorConfig, rng: random.Random,
                synthetic: SyntheticPredictorConfig | None = None) -> RequestOutcome:
    return DuchessRun(trace, config, rng, synthetic=synthetic).run()


def run_default_sc(trace: RequestTrace, config: OrchestratorConfig) -> RequestOutcome:
    return DefaultScRun(trace, config).run()


def run_short_mk(trace: RequestTrace, config: OrchestratorConfig) -> RequestOutcome:
    return ShortMkRun(trace, config).run()


def run_dynasor(trace: RequestTrace, config: OrchestratorConfig) -> RequestOutcome:
    return DynasorRun(trace, config).run()
