#!/usr/bin/env python
"""Standalone LaB-PQ (sssp_pq_*) timings on one GPU (exploration; profiles/pq_bench_r1.md).

n = 2^24 keys (uniform random 40-bit), batches of random ids (with duplicates).  Each call
is timed with CUDA events around the binding call (output tensors allocated beforehand);
calls that return a host value (extract count, size, theta, min) include their
synchronisation.  Device time per call: run under
`ncu --metrics gpu__time_duration.sum --csv` and sum the kernels of each call (scripts/pq_ncu.py).
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2105_06145_b200 as P  # noqa: E402


def timed(fn, reps=5):
    ts = []
    out = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


n = 1 << 24
g = torch.Generator(device="cuda").manual_seed(1)
keys = torch.randint(0, 1 << 40, (n,), dtype=torch.int64, device="cuda", generator=g)
pq = P.LabPQ(keys)
# first launches load the kernels (lazy module loading): warm every entry point once
pq.update(torch.arange(64, dtype=torch.int32, device="cuda"))
pq.size(), pq.select(8, seed=1), pq.select(8, seed=1, exact=True), pq.reduce_min(), pq.queue()
pq.extract(-1 & ((1 << 63) - 1), cap=n)  # drains the 64 warm-up ids
for batch in (1 << 16, 1 << 20, 1 << 23):
    ids = torch.randint(0, n, (batch,), dtype=torch.int32, device="cuda", generator=g)
    ms, _ = timed(lambda: pq.update(ids), reps=3)
    print(f"update  batch {batch:>9,}: {ms * 1e3:9.1f} us  ({batch / ms / 1e6:7.2f} G ids/s)", flush=True)
ms, sz = timed(lambda: pq.size())
print(f"size    |Q| = {sz:,}: {ms * 1e3:9.1f} us", flush=True)
for mode in (False, True):
    ms, th = timed(lambda: pq.select(1 << 18, seed=3, exact=mode))
    print(f"select  rho = 2^18 ({'exact' if mode else 'sampled'}): {ms * 1e3:9.1f} us", flush=True)
ms, mn = timed(lambda: pq.reduce_min())
print(f"reduce_min: {ms * 1e3:9.1f} us", flush=True)
th = pq.select(1 << 18, seed=3, exact=True)
outbuf = torch.empty(n, dtype=torch.int32, device="cuda")
ms, got = timed(lambda: pq.extract(th, cap=n, out=outbuf), reps=1)  # mutates Q: one timed call
print(f"extract theta = rho-th key: {ms * 1e3:9.1f} us, {got.numel():,} ids "
      f"(|Q| {sz:,} scanned: {sz / ms / 1e6:.2f} G ids/s)", flush=True)
ms, q = timed(lambda: pq.queue(out=outbuf), reps=3)
print(f"queue   ({q.numel():,} ids): {ms * 1e3:9.1f} us", flush=True)
pq.close()
