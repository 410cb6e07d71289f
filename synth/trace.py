"""C4: bursty synthetic online/offline trace -> hybrid batches (BASELINE.json configs[4]).

Shapes only (no arithmetic of the method).  Every parameter below is an
assumption stated in DESIGN.md §Inputs, because the paper gives no length
statistics; they are fixed here and not tuned afterwards.

* Online arrivals: Poisson with a sinusoidal envelope of burst factor 3
  (rate(t) = rho * base * (2 + sin(2 pi t / period)) / 2, so max/min = 3: "online
  request rates can vary by up to 3x within minutes").
  rho in {0, 0.5, 1, 2, 3}, base 2 req/s, period 120 s.
* Online prompts lognormal(median 1024, sigma 0.8) clipped [32, 8192];
  outputs lognormal(median 128, sigma 0.8) clipped [1, 1024].
* Offline backlog (always non-empty: HyGen fills residual capacity with
  offline work): arXiv-summarization-like prompts lognormal(median
  6144, sigma 0.5) clipped [1024, 16384], outputs median 256; plus MMLU-like
  requests in groups of 32 sharing a 1024-token prefix (suffix median 256).
* Batches come from a Sarathi-style composer (chunked prefill; Alg. 1
  order P:145-171): all running decodes (online first, at most 256), then
  prefill chunks, online before offline, up to the chunk budget C in
  {128, 256, 512, 1024, 2048}.  One iteration = 25 ms of trace time.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List

import numpy as np

from .configs import BatchSpec, Request

RHOS = (0.0, 0.5, 1.0, 2.0, 3.0)
CHUNKS = (128, 256, 512, 1024, 2048)
ITER_S = 0.025
BASE_QPS = 2.0
PERIOD_S = 120.0
MAX_DECODES = 256
MAX_CTX = 16384 + 1024


def _lognormal(rng, median, sigma, lo, hi):
    return int(min(hi, max(lo, round(math.exp(math.log(median) + sigma * rng.standard_normal())))))


@dataclass
class _Req:
    prompt: int
    output: int
    offline: bool
    group: int = -1
    prefix: int = 0
    done_prompt: int = 0
    done_out: int = 0
    rid: int = 0


class TraceSim:
    """Drives the composer; yields BatchSpecs (shapes of one hybrid iteration)."""

    def __init__(self, rho: float, chunk: int, seed: int, H_q=32, H_kv=8, d=128, B=16, offline_backlog=64):
        self.rng = np.random.default_rng(seed)
        self.rho, self.chunk = rho, chunk
        self.H_q, self.H_kv, self.d, self.B = H_q, H_kv, d, B
        self.t = self.rng.uniform(0, PERIOD_S)
        self.online: List[_Req] = []
        self.offline: List[_Req] = []
        self.next_id = 0
        self.next_group = 0
        self.backlog = offline_backlog
        self._refill_offline()

    def _new_id(self):
        self.next_id += 1
        return self.next_id

    def _refill_offline(self):
        while len(self.offline) < self.backlog:
            if self.rng.random() < 0.5:
                g = self.next_group
                self.next_group += 1
                for _ in range(32):
                    self.offline.append(_Req(1024 + _lognormal(self.rng, 256, 0.8, 16, 2048),
                                             _lognormal(self.rng, 256, 0.8, 1, 1024), True, g, 1024,
                                             rid=self._new_id()))
            else:
                self.offline.append(_Req(_lognormal(self.rng, 6144, 0.5, 1024, 16384),
                                         _lognormal(self.rng, 256, 0.8, 1, 1024), True, rid=self._new_id()))

    def _arrivals(self):
        rate = self.rho * BASE_QPS * (2.0 + math.sin(2 * math.pi * self.t / PERIOD_S)) / 2.0
        for _ in range(self.rng.poisson(rate * ITER_S)):
            self.online.append(_Req(_lognormal(self.rng, 1024, 0.8, 32, 8192),
                                    _lognormal(self.rng, 128, 0.8, 1, 1024), False, rid=self._new_id()))

    def step(self) -> BatchSpec:
        self._arrivals()
        reqs: List[Request] = []
        pool = self.online + self.offline
        # 1) running decodes, online first
        dec = [r for r in pool if r.done_prompt == r.prompt and r.done_out < r.output]
        dec = dec[:MAX_DECODES]
        for r in dec:
            reqs.append(Request(r.prompt + r.done_out, 1, r.offline, r.group, r.prefix, cid=r.rid))
        # 2) prefill chunks under the token budget, online before offline
        budget = self.chunk
        for r in pool:
            if budget <= 0:
                break
            if r.done_prompt < r.prompt:
                # a shared prefix already in the cache is credited (prefix caching)
                if r.group >= 0 and r.done_prompt == 0 and any(
                        o.group == r.group and o.done_prompt >= r.prefix for o in self.offline if o is not r):
                    r.done_prompt = r.prefix
                n = min(budget, r.prompt - r.done_prompt)
                reqs.append(Request(r.done_prompt, n, r.offline, r.group, r.prefix, cid=r.rid))
                r.done_prompt += n
                budget -= n
        for r in dec:
            r.done_out += 1
        self.online = [r for r in self.online if r.done_out < r.output]
        self.offline = [r for r in self.offline if r.done_out < r.output]
        self._refill_offline()
        self.t += ITER_S
        spec = BatchSpec(f"c4_rho{self.rho}_C{self.chunk}", self.H_q, self.H_kv, self.d, self.B, 0, reqs)
        return _share_fixup(spec)


def _share_fixup(spec: BatchSpec) -> BatchSpec:
    """Physically share a group's prefix blocks only among members whose cache
    already holds the whole prefix (c >= prefix); others keep private copies."""
    out = []
    for r in spec.requests:
        if r.group >= 0 and r.c < r.prefix_tokens:
            r = Request(r.c, r.n, r.offline, r.group, r.prefix_tokens, share=False, cid=r.cid)
        out.append(r)
    spec.requests = out
    return spec


def sweep(seed: int = 0, iters: int = 64, warm: int = 200, rhos=RHOS, chunks=CHUNKS, **shape) -> List[BatchSpec]:
    """len(rhos) * len(chunks) * iters batches (1,600 with the defaults)."""
    out = []
    for a, rho in enumerate(rhos):
        for b, C in enumerate(chunks):
            sim = TraceSim(rho, C, seed * 1000 + a * 10 + b, **shape)
            for _ in range(warm):
                sim.step()
            for _ in range(iters):
                spec = sim.step()
                if spec.requests:
                    out.append(spec)
    return out


def c4_batch(index: int, seed: int = 0, iters: int = 64, **shape) -> BatchSpec:
    """Batch number `index` of the C4 sweep (same order as ``sweep``): a named,
    regenerable test case (e.g. #219 of the Llama-3-8B sweep: a 49-token chunk at
    c = 10240 beside a 975-token chunk and 59 decodes)."""
    shape = {"H_q": 32, "H_kv": 8, "d": 128, **shape}
    return sweep(seed=seed, iters=iters, **shape)[index]
