"""Plain-Python / numpy restatement of the reference's probe + orchestration path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Used as the parity checker
for the CUDA path and, in bench.py, as the timed CPU reference ("port").
Citations are ``file:line`` under /root/reference/pkg/src/branchsim/.

The restatement is organised differently from the reference (a flat request
record plus pure step functions) but reproduces its observable behaviour:
RoundReports, RequestOutcomes, branch states and the random stream.
"""

from __future__ import annotations

import bisect
import math
import random
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# core.py

NO_ANSWER = ""                                    # core.py:19


def majority_vote(counts: dict[str, int]) -> str:
    """core.py:76-83 — highest count; ties -> smallest string."""
    if not counts:
        raise ValueError("no answers collected")
    top = max(counts.values())
    return min(a for a, n in counts.items() if n == top)


def at_least(frac: float, slots: int) -> int:
    """orchestrator.py:162-164."""
    return math.ceil(frac * slots - 1e-9)


def request_termination(counts: dict[str, int], consensus_frac: float,
                        coverage_frac: float, slots: int) -> str | None:
    """orchestrator.py:200-208 — consensus is checked before coverage."""
    if max(counts.values(), default=0) >= at_least(consensus_frac, slots):
        return "consensus"
    if sum(counts.values()) >= at_least(coverage_frac, slots):
        return "coverage"
    return None


# ---------------------------------------------------------------------------
# workload.py (templates are any object with natural_length, final_answer,
# probes, oracle_convergence, pred_probs — the reference's BranchTemplate
# works, as does a Tmpl below)

@dataclass
class Tmpl:
    natural_length: int
    final_answer: str
    probes: list = field(default_factory=list)
    oracle_convergence: int | None = None
    pred_probs: list | None = None


@dataclass
class Trace:
    id: str
    ground_truth: str
    prompt_tokens: int
    templates: list
    difficulty: int | None = None


def probe_answer(tmpl, position: int) -> str:
    """workload.py:82-94."""
    conv = tmpl.oracle_convergence
    if conv is not None and position >= conv:
        return tmpl.final_answer
    k = bisect.bisect_right([p[0] for p in tmpl.probes], position)
    return tmpl.probes[k - 1][1] if k > 0 else NO_ANSWER


def trace_prediction(tmpl, position: int) -> float:
    """workload.py:97-106."""
    if not tmpl.pred_probs:
        return 0.0
    k = bisect.bisect_right([p[0] for p in tmpl.pred_probs], position)
    return tmpl.pred_probs[k - 1][1] if k > 0 else 0.0


def synthetic_predict(converged: bool, rho: float, rng: random.Random) -> float:
    """predictor.py:328-335 — the uniform draw happens on every call."""
    u = rng.random()
    v = rho * (1.0 if converged else 0.0) + (1.0 - rho) * u
    return min(max(v, 0.0), 1.0)


def default_predictor(trace, rho: float):
    """orchestrator.py:211-224 make_correctness_predictor."""
    def predict(tmpl, position, rng):
        if tmpl.pred_probs:
            return trace_prediction(tmpl, position)
        return synthetic_predict(probe_answer(tmpl, position) == trace.ground_truth, rho, rng)
    return predict


# ---------------------------------------------------------------------------
# orchestrator.py rule primitives

def branch_out_weights(probs, temperature: float) -> list[float]:
    """orchestrator.py:177-185 (normaliser is the builtin sum: compensated on 3.12+)."""
    if len(probs) == 0:
        raise ValueError("no branch to duplicate")
    e = 1.0 / temperature
    raw = [min(max(p, 1e-6), 1.0) ** e for p in probs]
    z = sum(raw)
    return [x / z for x in raw]


def branch_out_sample(probs, temperature: float, rng: random.Random) -> int:
    """orchestrator.py:188-197."""
    w = branch_out_weights(probs, temperature)
    u = rng.random()
    acc = 0.0
    for i, x in enumerate(w):
        acc += x
        if u < acc:
            return i
    return len(w) - 1


def neumaier_sum(values) -> float:
    """CPython >= 3.12 builtin sum() over floats (Python/bltinmodule.c
    builtin_sum_impl); the reference's normaliser at orchestrator.py:184."""
    f, c = 0.0, 0.0
    for x in values:
        t = f + x
        if abs(f) >= abs(x):
            c += (f - t) + x
        else:
            c += (x - t) + f
        f = t
    if c and math.isfinite(c):
        f += c
    return f


# ---------------------------------------------------------------------------
# orchestrator.py — DUCHESS request state machine

ACTIVE, EARLY_TERMINATED, NATURAL_END, CAPPED, CANCELLED = (
    "active", "early_terminated", "natural_end", "capped", "cancelled")   # :35-40


@dataclass(frozen=True)
class Knobs:
    """orchestrator.py:62-96 OrchestratorConfig (validation restated)."""
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

    def __post_init__(self):
        bad = [
            (self.max_branches < 1, "max_branches must be >= 1"),
            (self.interval_tokens < 1, "interval_tokens must be >= 1"),
            (self.early_term_rounds < 1, "early_term_rounds must be >= 1"),
            (self.branch_out_temperature <= 0, "branch_out_temperature must be > 0"),
            (not 0.0 < self.consensus_frac <= 1.0, "consensus_frac must be in (0, 1]"),
            (not self.consensus_frac <= self.coverage_frac <= 1.0,
             "coverage_frac must be in [consensus_frac, 1]"),
            (self.token_cap < self.interval_tokens, "token_cap must be >= interval_tokens"),
            (self.probe_cost_tokens < 0, "probe_cost_tokens must be >= 0"),
        ]
        for cond, msg in bad:
            if cond:
                raise ValueError(msg)


@dataclass
class Branch:
    """orchestrator.py:99-125 BranchState."""
    branch_id: int
    template_index: int
    template: object
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


@dataclass
class Round:
    """orchestrator.py:149-159 RoundReport; actions are (kind, id, source)."""
    round_index: int
    decoding_branches: int
    max_chunk: int
    decode_tokens: int
    probes: int
    actions: list
    done: bool


@dataclass
class Outcome:
    """orchestrator.py:135-146 RequestOutcome (tally as a plain dict)."""
    tally: dict
    final: str
    termination_reason: str
    tokens_decode: int
    tokens_probe: int
    rounds: int


class DuchessRequest:
    """orchestrator.py:227-402 — RequestRun + DuchessRun restated."""

    def __init__(self, trace, knobs: Knobs, rng: random.Random, rho: float = 1.0,
                 predictor=None):
        self.trace, self.k, self.rng = trace, knobs, rng
        self.predict = predictor or default_predictor(trace, rho)
        self.counts: dict[str, int] = {}
        self.branches: list[Branch] = []
        self.tokens_decode = self.tokens_probe = self.rounds = 0
        self.outcome: Outcome | None = None
        self.next_template = 0
        for _ in range(min(knobs.max_branches, len(trace.templates))):   # :242-248
            self.spawn(0, None)

    @property
    def done(self) -> bool:
        return self.outcome is not None

    def spawn(self, offset: int, parent: Branch | None):                # :254-268
        if self.next_template >= len(self.trace.templates):
            return None
        j = self.next_template
        tmpl = self.trace.templates[j]
        b = Branch(branch_id=len(self.branches), template_index=j, template=tmpl,
                   offset_base=min(offset, tmpl.natural_length),
                   last_prediction=parent.last_prediction if parent else 0.5)
        self.next_template += 1
        self.branches.append(b)
        return b

    def active(self):
        return [b for b in self.branches if b.status == ACTIVE]

    def _vote(self, b: Branch, status: str, answer: str):               # :287-290
        b.status, b.final_answer = status, answer
        self.counts[answer] = self.counts.get(answer, 0) + 1

    def _probe(self, b: Branch) -> str:                                 # :281-285
        ans = probe_answer(b.template, b.position)
        b.probe_history.append((b.position, ans))
        self.tokens_probe += self.k.probe_cost_tokens
        return ans

    def _close(self, reason: str):                                      # :296-304
        self.outcome = Outcome(dict(self.counts), majority_vote(self.counts), reason,
                               self.tokens_decode, self.tokens_probe, self.rounds)

    def step(self) -> Round:                                            # :329-402
        if self.done:
            raise RuntimeError("request already terminated")
        k = self.k
        self.rounds += 1
        acts: list = []
        probes = decoding = max_chunk = dec_tokens = 0
        for b in self.active():                                         # phase 1
            room = min(b.template.natural_length, k.token_cap) - b.position
            n = max(0, min(k.interval_tokens, room))
            b.tokens_decoded += n
            self.tokens_decode += n
            if n:
                decoding += 1
                max_chunk = max(max_chunk, n)
                dec_tokens += n
            if b.position >= b.template.natural_length:
                self._vote(b, NATURAL_END, b.template.final_answer)
            elif b.position >= k.token_cap:
                probes += 1
                self._vote(b, CAPPED, self._probe(b))
        live = self.active()
        for b in live:                                                  # phase 2
            p = self.predict(b.template, b.position, self.rng)
            b.prediction_history.append(p)
            b.last_prediction = p
            b.streak = b.streak + 1 if p > k.early_term_threshold else 0
        for b in live:                                                  # phase 3
            if b.streak >= k.early_term_rounds:
                probes += 1
                self._vote(b, EARLY_TERMINATED, self._probe(b))
                acts.append(("terminate", b.branch_id, None))
            else:
                acts.append(("continue", b.branch_id, None))
        pool = self.active()                                            # phase 4
        while pool and len(pool) < k.max_branches and \
                self.next_template < len(self.trace.templates):
            src = pool[branch_out_sample([b.last_prediction for b in pool],
                                         k.branch_out_temperature, self.rng)]
            child = self.spawn(src.position, src)
            acts.append(("branch_out", child.branch_id, src.branch_id))
            pool.append(child)
        why = request_termination(self.counts, k.consensus_frac, k.coverage_frac,
                                  k.max_branches)                       # phase 5
        if why is not None:
            for b in self.active():
                b.status = CANCELLED
            self._close(why)
        elif not self.active():
            self._close("exhausted")
        return Round(self.rounds, decoding, max_chunk, dec_tokens, probes, acts, self.done)

    def run(self) -> Outcome:
        while not self.done:
            self.step()
        return self.outcome


# ---------------------------------------------------------------------------
# orchestrator.py:405-561 — baseline policies (restated on the same request base)

class _Baseline(DuchessRequest):
    def __init__(self, trace, knobs: Knobs):
        super().__init__(trace, knobs, rng=None, predictor=lambda *a: 0.0)

    def _round_start(self):
        if self.done:
            raise RuntimeError("request already terminated")
        self.rounds += 1

    def _advance(self, b: Branch):
        k = self.k
        room = min(b.template.natural_length, k.token_cap) - b.position
        n = max(0, min(k.interval_tokens, room))
        b.tokens_decoded += n
        self.tokens_decode += n
        return n


class DefaultScRequest(_Baseline):
    """orchestrator.py:405-435 — every branch runs to its end (or the cap)."""

    def step(self) -> Round:
        self._round_start()
        acts, probes, dec, mc, dt = [], 0, 0, 0, 0
        for b in self.active():
            n = self._advance(b)
            if n:
                dec, mc, dt = dec + 1, max(mc, n), dt + n
            if b.position >= b.template.natural_length:
                self._vote(b, NATURAL_END, b.template.final_answer)
            elif b.position >= self.k.token_cap:
                probes += 1
                self._vote(b, CAPPED, self._probe(b))
            else:
                acts.append(("continue", b.branch_id, None))
        if not self.active():
            self._close("exhausted")
        return Round(self.rounds, dec, mc, dt, probes, acts, self.done)


class ShortMkRequest(_Baseline):
    """orchestrator.py:438-516 — stop at the m-th finisher (lockstep cut)."""

    def __init__(self, trace, knobs: Knobs):
        if knobs.short_m > knobs.max_branches:
            raise ValueError(f"short_m ({knobs.short_m}) must not exceed max_branches "
                             f"({knobs.max_branches})")
        super().__init__(trace, knobs)
        self.finished = 0
        self.target = min(knobs.short_m, len(self.branches))

    def _finish_branch(self, b: Branch) -> int:
        if b.position >= b.template.natural_length:
            self._vote(b, NATURAL_END, b.template.final_answer)
            return 0
        self._vote(b, CAPPED, self._probe(b))
        return 1

    def step(self) -> Round:
        self._round_start()
        k = self.k
        plan = []
        for b in self.active():
            room = min(b.template.natural_length, k.token_cap) - b.position
            n = min(k.interval_tokens, room)
            plan.append((b, n, n == room))
        fins = sorted((n, b.branch_id, b) for b, n, f in plan if f)
        cut = None
        if self.finished + len(fins) >= self.target:
            cut = fins[self.target - self.finished - 1][0]
        probes = dec = mc = dt = 0
        for b, n, _f in plan:
            take = n if cut is None else min(n, cut)
            b.tokens_decoded += take
            self.tokens_decode += take
            if take > 0:
                dec, mc, dt = dec + 1, max(mc, take), dt + take
        if cut is None:
            for b, _n, f in plan:
                if f:
                    probes += self._finish_branch(b)
                    self.finished += 1
        else:
            done_n = self.finished
            for n, _bid, b in fins:
                if done_n < self.target and n <= cut:
                    probes += self._finish_branch(b)
                    done_n += 1
            self.finished = done_n
            for b in self.active():
                b.status = CANCELLED
            self._close("exhausted")
        if not self.done and not self.active():
            self._close("exhausted")
        return Round(self.rounds, dec, mc, dt, probes, [], self.done)


class DynasorRequest(_Baseline):
    """orchestrator.py:519-561 — probe every round, stop a branch once its last
    `dynasor_window` probe answers agree."""

    def __init__(self, trace, knobs: Knobs):
        if knobs.dynasor_window < 2:
            raise ValueError("dynasor_window must be >= 2")
        super().__init__(trace, knobs)

    def step(self) -> Round:
        self._round_start()
        win = self.k.dynasor_window
        probes = dec = mc = dt = 0
        for b in self.active():
            n = self._advance(b)
            if n:
                dec, mc, dt = dec + 1, max(mc, n), dt + n
            if b.position >= b.template.natural_length:
                self._vote(b, NATURAL_END, b.template.final_answer)
                continue
            if b.position >= self.k.token_cap:
                probes += 1
                self._vote(b, CAPPED, self._probe(b))
                continue
            ans = self._probe(b)
            probes += 1
            last = [a for _p, a in b.probe_history[-win:]]
            if len(last) == win and len(set(last)) == 1:
                self._vote(b, EARLY_TERMINATED, ans)
        if not self.active():
            self._close("exhausted")
        return Round(self.rounds, dec, mc, dt, probes, [], self.done)


BASELINES = {"default-sc": DefaultScRequest, "short-mk": ShortMkRequest,
             "dynasor": DynasorRequest}


# ---------------------------------------------------------------------------
# predictor.py — frozen MLP forward (restated; numpy f64)

def _gelu(x: np.ndarray) -> np.ndarray:
    return 0.5 * x * (1.0 + np.array([math.erf(v / math.sqrt(2.0)) for v in x]))


def mlp_forward(weights, activation):
    """predictor.py:126-151 — LN (population var, eps 1e-5) -> [W x + b -> BN ->
    act]* -> head -> clipped sigmoid (1-dim) or softmax."""
    x = np.asarray(activation, dtype=np.float64)
    if x.shape != (weights.input_dim,):
        raise ValueError(f"activation shape {x.shape} does not match expected "
                         f"({weights.input_dim},)")
    mu = x.mean()
    x = (x - mu) / math.sqrt(((x - mu) ** 2).mean() + 1e-5)
    if weights.ln_gain is not None:
        x = x * weights.ln_gain + weights.ln_bias
    for i, _ in enumerate(weights.layer_dims):
        x = weights.weights[i] @ x + weights.biases[i]
        if weights.bn_mean is not None:
            x = (x - weights.bn_mean[i]) / np.sqrt(weights.bn_var[i] + 1e-5)
            x = x * weights.bn_gain[i] + weights.bn_bias[i]
        x = np.maximum(x, 0.0) if weights.activations[i] == "relu" else _gelu(x)
    z = weights.weights[-1] @ x + weights.biases[-1]
    if weights.head_dim == 1:
        return z, np.clip(1.0 / (1.0 + np.exp(-z)), 1e-12, 1.0 - 1e-12)
    e = np.exp(z - z.max())
    return z, e / e.sum()


def pooled_linear_probe(window: np.ndarray, w: np.ndarray, b: float,
                        ln_gain: np.ndarray | None, ln_bias: np.ndarray | None):
    """Pool-then-probe restatement for the north-star's token window: the
    fp64 mean over T of the stored (bf16-rounded) values, then the linear
    probe of predictor.py:134-148. Returns (logit, prob)."""
    m = np.asarray(window, dtype=np.float64).mean(axis=0)
    mu = m.mean()
    z = (m - mu) / math.sqrt(((m - mu) ** 2).mean() + 1e-5)
    if ln_gain is not None:
        z = z * ln_gain + ln_bias
    logit = float(w @ z + b)
    return logit, min(max(1.0 / (1.0 + math.exp(-logit)), 1e-12), 1.0 - 1e-12)


# ---------------------------------------------------------------------------
# predictor.py — difficulty prediction; scheduler.py — ordering

CONFUSION = (
    (0.40, 0.25, 0.16, 0.12, 0.07),
    (0.18, 0.42, 0.20, 0.13, 0.07),
    (0.08, 0.18, 0.40, 0.22, 0.12),
    (0.04, 0.10, 0.22, 0.42, 0.22),
    (0.03, 0.06, 0.10, 0.35, 0.46),
)                                                                 # predictor.py:353-359


def confused_level(true_level: int, rng: random.Random, matrix=CONFUSION) -> int:
    """predictor.py:376-386."""
    u = rng.random()
    acc = 0.0
    for lvl, p in enumerate(matrix[true_level - 1], start=1):
        acc += p
        if u < acc:
            return lvl
    return 5


def service_order(entries) -> list[int]:
    """Repeated scheduler.py:60-96 next_request pops (easiest-first) over one
    snapshot where every entry is eligible: the order of (level, arrival,
    order) keys. ``entries`` is a list of (level, arrival, order)."""
    pending = list(range(len(entries)))
    out = []
    while pending:
        best = min(pending, key=lambda i: entries[i])
        pending.remove(best)
        out.append(best)
    return out


# ---------------------------------------------------------------------------
# workload.py:317-413 — synthetic workload generation (restated; the same
# random-call sequence, so a seed reproduces the reference's workload)

@dataclass(frozen=True)
class GenParams:
    level_median_tokens: tuple = (340, 460, 640, 840, 1180)
    length_sigma: float = 0.30
    level_correct_prob: tuple = (0.85, 0.78, 0.70, 0.62, 0.52)
    convergence_range: tuple = (0.3, 0.7)
    templates_per_request: int = 10
    distractor_count: int = 6
    probe_stride: int = 16
    prompt_token_range: tuple = (60, 200)
    level_mix: tuple | None = None
    token_cap: int = 4096
    min_length: int = 16


def generate(params: GenParams, n_requests: int, seed: int) -> list[Trace]:
    rng = random.Random(seed)
    out = []
    for i in range(n_requests):
        level = (rng.randint(1, 5) if params.level_mix is None
                 else rng.choices((1, 2, 3, 4, 5), weights=params.level_mix, k=1)[0])
        truth = str(rng.randrange(100, 100000))
        wrong: list[str] = []
        while len(wrong) < params.distractor_count:
            cand = str(rng.randrange(100, 100000))
            if cand != truth and cand not in wrong:
                wrong.append(cand)
        tmpls = []
        for _ in range(params.templates_per_request):
            med = params.level_median_tokens[level - 1]
            n = int(round(med * math.exp(params.length_sigma * rng.gauss(0.0, 1.0))))
            n = max(params.min_length, min(n, params.token_cap))
            final = truth if rng.random() < params.level_correct_prob[level - 1] \
                else rng.choice(wrong)
            conv = max(1, int(round(rng.uniform(*params.convergence_range) * n)))
            probes = [(at, rng.choice(wrong))
                      for at in range(params.probe_stride, conv, params.probe_stride)]
            tmpls.append(Tmpl(n, final, probes, conv))
        out.append(Trace(f"r{i:05d}", truth, rng.randint(*params.prompt_token_range),
                         tmpls, level))
    return out
