"""Build variant libraries for A/B timing (tuning aid).

  python scripts/ab_build.py name1 "-DX=1 -DY=0" name2 "-DX=0" ...
writes build/ab/<name>.so; scripts/ab_run.sh times each on the GPU.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, os.getcwd())
from paper_2507_01522_b200 import _build as B  # noqa: E402

out = Path("build/ab")
out.mkdir(parents=True, exist_ok=True)
pairs = list(zip(sys.argv[1::2], sys.argv[2::2]))


def one(pair):
    name, flags = pair
    objs = []
    for src in B._sources():
        o = out / f"{name}_{src.stem}.o"
        subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *flags.split(), "-c", str(src), "-o", str(o)], check=True,
                       capture_output=True)
        objs.append(str(o))
    subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(out / f"{name}.so"),
                    *objs], check=True)
    return name


with ThreadPoolExecutor(len(pairs)) as ex:
    for n in ex.map(one, pairs):
        print("built", out / f"{n}.so")
