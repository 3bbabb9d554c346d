"""Build the sm_100a C-ABI library in-tree (no JIT cache, travels with gpurun).

    python paper_2108_07126_b200/build.py        # or __graft_entry__.build()

(run it as a file: importing the package first would load the old library)

Produces ``paper_2108_07126_b200/libsliceprop_b200.so`` from
``csrc/engine.cu`` (kernels + C ABI) and ``csrc/plan.cpp`` (host plan), with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and a static cudart so
the library loads on machines without a GPU (for the CPU test tier).
"""

from __future__ import annotations

import os
import re
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsliceprop_b200.so")
SOURCES = [os.path.join(CSRC, "engine.cu"), os.path.join(CSRC, "batch.cu"),
           os.path.join(CSRC, "su2.cu"), os.path.join(CSRC, "plan.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("kernels.cuh", "kernels_tc.cuh", "kernels_ps.cuh", "kernels_ps3.cuh", "kernels_ps3g.cuh", "kernels_apply.cuh", "kernels_d8.cuh", "kernels_batch.cuh", "kernels_f32.cuh", "kernels_su2.cuh",
                                                  "internal.h")] + [
    os.path.join(ROOT, "include", "sliceprop_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = OUT,
          defines: tuple = ()) -> str:
    """Build the library (``out``/``defines``: instrumented variants for tools/)."""
    if not force and up_to_date(out):
        return out
    # one nvcc per translation unit, in parallel, then one link step
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    common = [nvcc(), *[f for f in NVCC_FLAGS if f != "-shared"],
              *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    tmpdir = tempfile.mkdtemp(prefix="spbuild")
    objs = [os.path.join(tmpdir, os.path.basename(src) + ".o") for src in SOURCES]

    def compile_one(args):
        src, obj = args
        cmd = [*common, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return r.returncode, " ".join(cmd) + "\n" + r.stdout + r.stderr

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, zip(SOURCES, objs)))
    log = "".join(r[1] for r in results)
    rc = max(r[0] for r in results)
    if rc == 0:
        cmd = [nvcc(), "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", *objs,
               "-o", out + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log += " ".join(cmd) + "\n" + r.stdout + r.stderr
        rc = r.returncode
    shutil.rmtree(tmpdir, ignore_errors=True)

    class res:  # noqa: N801  (keeps the checks below unchanged)
        returncode = rc
    with open(os.path.join(HERE, "build.log" if out == OUT else "build_variant.log"), "w") as fh:
        fh.write(log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{log[-4000:]}")
    if any(int(n) > 0 for n in re.findall(r"(\d+) bytes spill stores", log)):
        print("warning: register spills in the sm_100a build (see build.log)", file=sys.stderr)
    os.replace(out + ".tmp", out)
    if verbose:
        print(log)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
