"""Build libsssp.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

The round-loop kernel template (csrc/loop.cuh) is instantiated per (policy, bidirectional,
fusion) triple: csrc/inst.cu is compiled once per triple with -DINST_POL/-DINST_BIDIR/-DINST_FUSE
(plus UNIT_DEFINES), in parallel with the other translation units, and everything is linked
into one shared library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsssp.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
POLICIES = 5  # SSSP_RHO .. SSSP_DELTA_STEPPING (include/sssp.h)


# Unit-specific tuning constants (the constants of csrc/loop.cuh are compile-time): the
# rho kernels without fusion relax more arcs per lane per step (more gathers in flight; the
# fusion kernels spill with it).  Before deferred WriteMins, 6 arcs: rmat24 rho = 2^18
# -2.6 %, 2^21 -6 % against 4.
# The segment hint in phase B (forward scan instead of a binary search per descriptor)
# helps BF / Delta* by ~2 %; the rho unit kept the binary search while the next descriptor
# lived in registers (round 1), and gains 0.3-1.2 % from the hint since it moved to cp.async.
# With deferred WriteMins the rho unit does best at 5 arcs per lane (A/B against 6:
# rmat24 rho = 2^18 -2.9 %, 2^17 -3.1 %, rmat20 -4 %; 7 arcs: +2 %).
# The Delta* unit likewise (rmat24 -1.6 %, rmat20 -2.4 %); BF stays at 4 (+8-12 % with 5).
# Phase B with dynamic per-CTA item assignment (SSSP_DYN_B) helps the rho and Delta* units
# (rmat24 Delta* -3.1 %, rmat20 -3.4 %, rho -0.7 / -1 %) and costs BF 8-12 % (round 2 A/B).
# The static order's next descriptor by cp.async (SSSP_NEXT_SMEM) lost 4.6 % on BF, which keeps
# it in registers.
UNIT_DEFINES = {(0, 0, 0): ["-DSSSP_ARCS=5", "-DSSSP_DYN_B=1"],
                (1, 0, 0): ["-DSSSP_ARCS=5", "-DSSSP_DYN_B=1"],
                (2, 0, 0): ["-DSSSP_NEXT_SMEM=0"]}


def units(unit_defines=None):
    """(name, source, extra defines) for every object file of the library."""
    ud = {k: list(v) for k, v in UNIT_DEFINES.items()}
    for k, v in (unit_defines or {}).items():
        ud[k] = ud.get(k, []) + list(v)
    out = [(os.path.splitext(os.path.basename(s))[0], s, []) for s in sorted(glob.glob(os.path.join(CSRC, "*.cu")))
           if os.path.basename(s) != "inst.cu"]
    inst = os.path.join(CSRC, "inst.cu")
    for pol in range(POLICIES):
        for bidir in (0, 1):
            for fuse in (0, 1):
                out.append((f"inst_{pol}_{bidir}_{fuse}", inst,
                            [f"-DINST_POL={pol}", f"-DINST_BIDIR={bidir}", f"-DINST_FUSE={fuse}"]
                            + ud.get((pol, bidir, fuse), [])))
    return out


def deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(HERE, "..", "include", "sssp.h"),
                                                           os.path.abspath(__file__)]  # UNIT_DEFINES live here


def up_to_date(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = True, out: str = OUT, defines=(), unit_defines=None,
          only_units=None) -> str:
    """Compile every translation unit (in parallel) and link the shared library.
    defines: tuning variants for every unit, e.g. SSSP_ARCS=4; unit_defines: {(pol, bidir,
    fuse): ["-DNAME=VAL", ...]} added to one unit (both written to a separate `out`).
    only_units: names (e.g. {"inst_0_0_0", "pq"}) to compile; the other objects are taken
    from the default build's object directory (A/B variants of one unit in seconds)."""
    if not force and out == OUT and not defines and not unit_defines and up_to_date():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    tag = os.path.splitext(os.path.basename(out))[0]
    # object files live outside the tree (they are ~40 MB per variant; only the linked
    # .so travels with the repo snapshot)
    objdir = os.path.join(os.environ.get("SSSP_BUILD_DIR", os.path.join(tempfile.gettempdir(), "sssp_build")), tag)
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_one(u):
        name, src, extra = u
        obj = os.path.join(objdir, name + ".o")
        if only_units is not None and name not in only_units:
            import shutil

            shutil.copyfile(os.path.join(os.path.dirname(objdir), "libsssp", name + ".o"), obj)
            return name, obj, ["(copied from the default build)"], subprocess.CompletedProcess([], 0, "", "")
        cmd = [nvcc, *NVCC_FLAGS, *dflags, *extra, "-c", "-o", obj, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return name, obj, cmd, res

    jobs = int(os.environ.get("SSSP_BUILD_JOBS", str(os.cpu_count() or 4)))
    with ThreadPoolExecutor(max_workers=max(1, jobs)) as ex:
        results = list(ex.map(compile_one, units(unit_defines)))
    log_path = os.path.join(HERE, "build.log" if out == OUT else os.path.basename(out) + ".log")
    with open(log_path, "w") as log:
        for name, obj, cmd, res in results:
            log.write(f"### {name}: {' '.join(cmd)}\n{res.stdout}{res.stderr}\n")
    failed = [(n, r) for n, _, _, r in results if r.returncode != 0]
    if failed:
        for n, r in failed:
            sys.stderr.write(f"--- {n}\n{r.stdout}{r.stderr}")
        raise RuntimeError(f"nvcc failed for {[n for n, _ in failed]}; see {log_path}")
    link = [nvcc, *ARCH, "-shared", "-o", out, *[obj for _, obj, _, _ in results]]
    if verbose:
        print(" ".join(link), flush=True)
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"link failed ({res.returncode})")
    return out


if __name__ == "__main__":
    # python build.py [--force] [--out lib.so] [-DNAME=VAL ...] [--unit P,B,F:NAME=VAL ...] [--only inst_0_0_0,...]
    args = sys.argv[1:]
    out = OUT
    if "--out" in args:
        out = os.path.abspath(args[args.index("--out") + 1])
    ud = {}
    for i, a in enumerate(args):
        if a == "--unit":
            key, d = args[i + 1].split(":")
            ud.setdefault(tuple(int(x) for x in key.split(",")), []).append("-D" + d)
    only = None
    if "--only" in args:
        only = set(args[args.index("--only") + 1].split(","))
    build(force="--force" in args, out=out, defines=[a[2:] for a in args if a.startswith("-D")], unit_defines=ud,
          only_units=only)
