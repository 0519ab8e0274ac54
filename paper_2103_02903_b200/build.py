"""In-tree build of libmrlbm_b200.so for sm_100a (nvcc; no JIT cache)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "mrlbm_step.cu"), os.path.join(HERE, "csrc", "host_configs.cpp")]
OUT = os.path.join(HERE, "libmrlbm_b200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                      # bit parity with the oracle: no FMA contraction
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-shared",
]


def build(verbose=False):
    gen = os.path.join(HERE, "csrc", "stream_gen.cuh")
    gen_src = [os.path.join(HERE, "csrc", "gen_stream.py"), os.path.join(HERE, "csrc", "collide_patterns.json")]
    # regenerate the unrolled table code whenever its generator (or its input) is newer
    if not os.path.exists(gen) or any(os.path.getmtime(p) > os.path.getmtime(gen) for p in gen_src if os.path.exists(p)):
        subprocess.run([sys.executable, gen_src[0]], check=True)
    deps = SRC + [os.path.join(HERE, "csrc", "mrlbm_internal.h"), gen, os.path.join(ROOT, "include", "mrlbm_gpu.h")]
    if os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(p) for p in deps):
        return OUT
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-o", OUT] + SRC
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
