"""In-tree build of libmrlbm_b200.so for sm_100a (nvcc; no JIT cache).

Each translation unit is compiled to an object under csrc/_obj/ (only when it or a
header it includes is newer), the units in parallel, then linked.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "_obj")
OUT = os.path.join(HERE, "libmrlbm_b200.so")
GEN = os.path.join(CSRC, "stream_gen.cuh")
HEADERS = [os.path.join(CSRC, "mrlbm_internal.h"), os.path.join(ROOT, "include", "mrlbm_gpu.h")]
# source -> extra dependencies
UNITS = {
    os.path.join(CSRC, "mrlbm_step.cu"): [GEN],
    os.path.join(CSRC, "mrlbm_step3d.cu"): [],
    os.path.join(CSRC, "host_configs.cpp"): [],
}
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                      # bit parity with the oracle: no FMA contraction
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
]


def _stale(target, deps):
    return not os.path.exists(target) or any(os.path.getmtime(p) > os.path.getmtime(target) for p in deps)


def build(verbose=False):
    gen_src = [os.path.join(CSRC, "gen_stream.py"), os.path.join(CSRC, "collide_patterns.json")]
    # regenerate the unrolled table code whenever its generator (or its input) is newer
    if _stale(GEN, [p for p in gen_src if os.path.exists(p)]):
        subprocess.run([sys.executable, gen_src[0]], check=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJ, exist_ok=True)
    jobs, objs = [], []
    for src, extra in UNITS.items():
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, [src] + HEADERS + extra):
            jobs.append([nvcc] + NVCC_FLAGS + ["-c", "-o", obj, src])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        list(ex.map(run, jobs))
    if jobs or _stale(OUT, objs):
        run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", OUT] + objs)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
