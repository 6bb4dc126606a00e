"""Steady-state C2 launches of one mode (argv[1]: fused | nodecide | k1) for
ncu captures."""
import sys
import torch
sys.path.insert(0, ".")
from tools.step_probe import engine, bank, slabs, logit, rows, Scorer, _lib  # noqa: E402

mode = sys.argv[1]
eng = engine()
if mode in ("fused", "nodecide"):
    eng.begin_fused()
    for i in range(12):
        if mode == "nodecide" and i == 8:
            eng.policy.flags |= _lib.FLAG_PROFILE_NO_DECIDE
        eng.step_fused(slabs[i % 4], bank, logit.view(-1))
else:
    sc = Scorer(bank, rows)
    probs = eng.probs.view(rows, 1)
    eng.advance()
    for i in range(12):
        sc.score_active(slabs[i % 4], logit, probs, eng)
        eng.round()
torch.cuda.synchronize()
