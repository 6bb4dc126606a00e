"""The serving loop: probe scoring + orchestration rounds over request shards.

One GPU serves a pool of requests through ``S`` independent request shards
(``BatchedDuchess`` engines over one packed pool, each with its own slice of
the service queue), each stepping on its own CUDA stream. A round of a shard
is two or three launches:

  ``Scorer.score_active``  K1: pooled LayerNorm + linear probe(s) over the
                           survivors of the round in flight (the device-side
                           active list), probabilities by branch slot;
  ``BatchedDuchess.round`` K2: decide the round (orchestrator.py:357-402),
                           refill finished slots from the queue and advance
                           every slot into the next round (:344-355);
  ``PagedKVCache.round``   K3 (optional, ``kv=``): the round's forks share
                           their root's KV blocks copy-on-write, ended
                           branches release theirs, decoding branches grow
                           (kvfork.py, duchess_kv_round). It runs right after
                           its round and releases the next round's scorer,
                           which streams beside it (``kv_mode="lead"``), so it
                           is off the scorer -> round chain.

Requests never interact (reference SPEC.md:295), so shards are exact: each
request's rounds depend only on its own state, RNG stream and activation
windows, not on which shard or slot serves it. Two shards on one GPU keep one
shard's latency-bound round kernel beside the other shard's HBM-bound scorer.
The same class is the per-rank engine of the multi-GPU path
(``distributed.run_sharded``). This is the loop ``bench.py`` times.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .engine import BatchedDuchess, pack_pool
from .kvfork import PagedKVCache
from .mlp_probe import MlpProbeBank, MlpScorer
from .probe import Scorer, fill_windows


class ShardedEngine:
    """S request shards of one request pool on one GPU.

    traces / config / seeds: the pool (RequestTrace-likes, OrchestratorConfig,
    per-request seeds as for DuchessRun's rng). bank: ProbeBank (L linear
    probes of width H, K1) or MlpProbeBank (the paper's MLP probe per layer on
    the tensor cores, T = 1). n_slots: request slots in total (split evenly over the shards).
    queue: service order of pool indices (default: pool order); shard k takes
    queue[k::S]. T, dtype: the activation window per branch-step. kv: None,
    or PagedKVCache keyword arguments (block_tokens, blocks_per_slot,
    kv_bytes_per_token) for a paged KV cache per shard, updated every round.
    """

    def __init__(self, traces, config, seeds, bank, *, n_slots: int, shards: int = 2,
                 queue=None, cycle: bool = False, T: int = 1, dtype=torch.bfloat16,
                 device="cuda", combine: int | None = None, n_buffers: int = 1,
                 packed=None, kv: dict | None = None, kv_mode: str | None = None):
        _lib.require_cuda()
        if shards < 1 or n_slots % shards:
            raise ValueError(f"{shards} shards must evenly divide the {n_slots} request slots")
        self.device = torch.device(device)
        # Where K3 (the paged-KV update of a round) runs:
        #   "lead" (default): its own launch right after the round, releasing the
        #       next round's scorer at once; the scorer streams beside it
        #       (SCORE_NO_INPUT_WAIT) and completes after it, so the round after
        #       sees it done: K3 is off the scorer -> round chain;
        #   "overlap": its own launch right after the next round's scorer,
        #       beside it; the next round waits for it (measured 0-4% slower at
        #       C2; DUCHESS_KV_MODE=overlap, for measurement).
        self.kv_mode = kv_mode or os.environ.get("DUCHESS_KV_MODE", "lead")
        if self.kv_mode not in ("lead", "overlap"):
            raise ValueError(f"unknown kv_mode {self.kv_mode!r}")
        self.bank = bank
        self.S, self.L, self.T, self.H = shards, bank.L, T, bank.H
        self.dtype = dtype
        self.C = int(config.max_branches)
        self.Rs = n_slots // shards
        self.rows = self.Rs * self.C
        P = len(traces)
        queue = list(range(P)) if queue is None else list(queue)
        self.packed = packed if packed is not None else pack_pool(traces, seeds, self.device)
        combine = (1 if bank.L > 1 else 0) if combine is None else combine
        self.shards = []
        for k in range(shards):
            eng = BatchedDuchess(traces, config, seeds, n_slots=self.Rs,
                                 pred_source=_lib.PRED_DEVICE, queue=queue[k::shards],
                                 cycle=cycle, n_layers=bank.L, combine=combine,
                                 device=self.device, packed=self.packed)
            acts = [torch.zeros((self.rows, bank.L, T, bank.H), dtype=dtype, device=self.device)
                    for _ in range(n_buffers)]
            scorer = (MlpScorer(bank) if isinstance(bank, MlpProbeBank)
                      else Scorer(bank, self.rows * bank.L))
            self.shards.append(dict(
                eng=eng, scorer=scorer, acts=acts,
                logit=torch.zeros((self.rows, bank.L), dtype=torch.float32, device=self.device),
                stream=torch.cuda.Stream(self.device), ev=[],
                kv=None if kv is None else PagedKVCache(eng, **kv), kv_pending=False,
                kv_led=False))
        self.started = False

    @property
    def engines(self):
        return [sh["eng"] for sh in self.shards]

    # ------------------------------------------------------------------
    def fork(self):
        """Shard streams wait for the caller's (current) stream."""
        cur = torch.cuda.current_stream(self.device)
        for sh in self.shards:
            sh["stream"].wait_stream(cur)

    def join(self):
        """The caller's (current) stream waits for every shard."""
        cur = torch.cuda.current_stream(self.device)
        for sh in self.shards:
            cur.wait_stream(sh["stream"])

    def flush_kv(self):
        """Apply the KV update still pending for the latest round (kv_mode
        "overlap" defers it to run beside the next round's scorer)."""
        for sh in self.shards:
            if sh["kv_pending"]:
                with torch.cuda.stream(sh["stream"]):
                    sh["kv"].round()
                sh["kv_pending"] = False

    def begin(self):
        """Refill every slot and run phase 1 of the first round."""
        self.fork()
        for sh in self.shards:
            with torch.cuda.stream(sh["stream"]):
                sh["eng"].advance()
                if sh["kv"] is not None and self.kv_mode != "overlap":
                    sh["kv"].round()                        # K3 of the first phase 1
            sh["kv_pending"] = sh["kv"] is not None and self.kv_mode == "overlap"
            sh["kv_led"] = False
        self.started = True

    def step(self, i: int = 0, *, fill=None, timed: bool = False, after_round=None,
             before_round=None):
        """One round of every shard, each on its stream (no host sync).

        i: round counter (selects activation buffer i % n_buffers).
        fill(k, eng, acts): optional window source, called on shard k's stream
            before scoring (e.g. the keyed synthetic fill of the round's
            survivors, or a host upload); by default the buffer is used as is.
        timed: bracket the scorer launch with CUDA events on the shard stream.
        after_round(k, eng): optional hook on the shard stream after round() (and,
            with kv_mode "lead", after K3 of the round; with "overlap" K3 of the
            round is applied during the next step: flush_kv() first).
        before_round(k, eng): optional hook on the shard stream right before
            round() — after K3 of the previous round completed.
        """
        if not self.started:
            self.begin()
        for k, sh in enumerate(self.shards):
            st = sh["stream"]
            with torch.cuda.stream(st):
                eng = sh["eng"]
                acts = sh["acts"][i % len(sh["acts"])]
                if fill is not None:
                    fill(k, eng, acts)
                if timed:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                # kv "lead": the launch before this scorer is this shard's K3,
                # which started only after the round that produced the inputs
                # here completed (hooks in between launch ordinary kernels,
                # which complete before the scorer starts): the scorer streams
                # at once, beside K3, and completes after it
                if sh["kv_led"] and not timed and isinstance(sh["scorer"], Scorer):
                    sh["scorer"].score_active(acts, sh["logit"],
                                              eng.probs.view(self.rows, self.L), eng,
                                              no_input_wait=True)
                else:
                    sh["scorer"].score_active(acts, sh["logit"],
                                              eng.probs.view(self.rows, self.L), eng)
                sh["kv_led"] = False
                if timed:
                    e1.record(st)
                    sh["ev"].append((e0, e1))
                if sh["kv_pending"]:
                    # K3 of the previous round, overlapped with this round's
                    # scorer (which reads only the active list and windows);
                    # it completes after the scorer, before this round()
                    sh["kv"].round(overlap=not timed)
                    sh["kv_pending"] = False
                if before_round is not None:
                    before_round(k, eng)
                eng.round()
                if sh["kv"] is not None:
                    if self.kv_mode == "lead":
                        sh["kv"].round(lead=True)
                        sh["kv_led"] = True
                    else:
                        sh["kv_pending"] = True
                if after_round is not None:
                    after_round(k, eng)

    def run(self, max_rounds: int = 100000, fill=None, after_round=None,
            before_round=None) -> int:
        """Serve the queues to completion (non-cycling pools). Returns rounds."""
        if not self.started:
            self.begin()
        for i in range(max_rounds):
            self.step(i, fill=fill, after_round=after_round, before_round=before_round)
            if i % 8 == 7:
                self.flush_kv()
                self.join()
                if self.all_done():
                    return i + 1
        self.flush_kv()
        self.join()
        if not self.all_done():
            raise RuntimeError(f"requests still running after {max_rounds} rounds")
        return max_rounds

    # ------------------------------------------------------------------
    def all_done(self) -> bool:
        torch.cuda.synchronize(self.device)
        return all(sh["eng"].all_done() for sh in self.shards)

    def counters(self):
        return sum(sh["eng"].counters() for sh in self.shards)

    def outcomes(self) -> dict:
        """{pool index: outcome dict} over every shard (finished requests)."""
        out = {}
        for sh in self.shards:
            for p, o in enumerate(sh["eng"].outcomes()):
                if o is not None:
                    out[p] = o
        return out

    def kv_counters(self) -> dict | None:
        """Summed PagedKVCache counters over the shards (None without kv)."""
        if self.shards[0]["kv"] is None:
            return None
        tot: dict = {}
        for sh in self.shards:
            for k, v in sh["kv"].counters().items():
                tot[k] = tot.get(k, 0) + v
        tot["peak_blocks_per_slot"] = max(
            int(sh["kv"].t["arena"].view(-1, 4)[:, 3].max()) for sh in self.shards)
        return tot

    def scorer_events(self):
        return [ev for sh in self.shards for ev in sh["ev"]]


def keyed_fill(seed: int):
    """Window source keyed by (pool request, template, position): the
    synthetic stand-in for the LLM's activations. oracle/activations.py
    regenerates the same windows bit for bit on the CPU, and a request's
    windows do not depend on its slot, shard or rank."""
    def fill(_k, eng, acts):
        t = eng.t
        fill_windows(acts, seed, t["row_req"], t["row_tmpl"], t["row_pos"], t["row_mask"])
    return fill
