#!/usr/bin/env python
"""Hardware ceilings of the relax access pattern on rmat24 (exploration; see relax_bench.cu)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "scripts", "librelaxbench.so"))
lib.relax_bench.restype = ctypes.c_float
lib.relax_bench.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 5 + [
    ctypes.c_int]
name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
g = gen.make(name)
idx = torch.from_numpy(g.indices).cuda()
w = torch.from_numpy(g.weights.view("int32")).cuda()
dist = torch.randint(0, 1 << 40, (g.n,), dtype=torch.int64, device="cuda")
key = torch.randint(0, 1 << 30, (g.n,), dtype=torch.int32, device="cuda")
out = torch.zeros(4, dtype=torch.int64, device="cuda")
m = g.m
names = {0: "stream idx+w", 1: "+gather u64", 2: "+gather u32", 3: "+gather u64+atomicMin", 4: "+blind RED.MIN u64",
         5: "+blind RED.MIN u32"}
modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 4, 5]
for mode in modes:
    for arcs in (4, 8, 16):
        for bpsm in (2, 4):
            blocks = 148 * bpsm
            if mode == 3:
                dist.copy_(torch.randint(0, 1 << 40, (g.n,), dtype=torch.int64, device="cuda"))
            ms = lib.relax_bench(mode, arcs, blocks, m, idx.data_ptr(), w.data_ptr(), dist.data_ptr(), key.data_ptr(),
                                 out.data_ptr(), 5)
            print(f"{name} {names[mode]:24s} arcs/thr {arcs:2d} grid {blocks}x512: {ms:7.3f} ms  "
                  f"{m / ms / 1e6:7.1f} Garcs/s  stream {8 * m / ms / 1e6:7.1f} GB/s  "
                  f"'touched' {16 * m / ms / 1e6:7.1f} GB/s", flush=True)
