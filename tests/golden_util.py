"""Helpers shared by the oracle (CPU) and CUDA (GPU) parity tests: load the
golden fixtures made from the reference and rebuild their inputs without
needing /root/reference (the GPU box does not have it)."""

from __future__ import annotations

import hashlib
import json
import math
from functools import lru_cache
from pathlib import Path

from oracle import port

GOLDEN = Path(__file__).resolve().parent / "golden"
STATUS = {0: "active", 1: "early_terminated", 2: "natural_end", 3: "capped", 4: "cancelled"}
KIND = {1: "continue", 2: "terminate", 3: "branch_out"}


@lru_cache(maxsize=None)
def load(name: str):
    return json.loads((GOLDEN / name).read_text())


def fx(h: str) -> float:
    return float.fromhex(h)


def workload_digest(requests) -> str:
    h = hashlib.sha256()
    for r in requests:
        h.update(json.dumps([r.id, r.ground_truth, r.prompt_tokens, r.difficulty,
                             [[t.natural_length, t.final_answer, [list(p) for p in t.probes],
                               t.oracle_convergence,
                               None if t.pred_probs is None else
                               [[a, float(p).hex()] for a, p in t.pred_probs]]
                              for t in r.templates]]).encode())
    return h.hexdigest()


def gen_params(d: dict) -> port.GenParams:
    d = {k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()}
    return port.GenParams(**d)


def case_traces(case) -> list:
    if "traces" in case:
        out = []
        for rid, gt, pt, diff, tmpls in case["traces"]:
            ts = [port.Tmpl(n, fin, [tuple(p) for p in probes], conv,
                            None if pp is None else [(a, fx(p)) for a, p in pp])
                  for n, fin, probes, conv, pp in tmpls]
            out.append(port.Trace(rid, gt, pt, ts, diff))
        return out
    return port.generate(gen_params(case["params"]), case["n"], case["workload_seed"])


def case_knobs(case) -> port.Knobs:
    cfg = dict(case["config"])
    cfg["early_term_threshold"] = fx(cfg["early_term_threshold"])
    return port.Knobs(**cfg)


def report_tuple(r):
    """Normalise a golden report list to the engine's tuple form."""
    rnd, dec, mc, dt, pr, acts, done = r
    return (rnd, dec, mc, dt, pr,
            [(KIND[k], b, None if s < 0 else s) for k, b, s in acts], bool(done))


def port_report_tuple(rep: "port.Round"):
    return (rep.round_index, rep.decoding_branches, rep.max_chunk, rep.decode_tokens,
            rep.probes, [tuple(a) for a in rep.actions], rep.done)


def is_inf(x: float) -> bool:
    return math.isinf(x)
