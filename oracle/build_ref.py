"""Build the reference's own compiled stepping kernel into oracle/_ref/.

TEST INFRASTRUCTURE.  Compiles /root/reference/pkg/src/voltyard/backends/
_kernel.pyx where it lies (Cython -> C in a /tmp scratch dir, then gcc with
the reference's flags -O3 -ffp-contract=off, pkg/setup.py:18-28).  Only the
resulting extension module lands in oracle/_ref/ (git-ignored, travels to the
GPU box).  No reference source is copied into the repository.

The module exposes CySimCore(tables, states, outs); oracle/harness.py drives
it with duck-typed table/state objects, so the reference's real kernel runs
on the GPU box without the rest of the voltyard package.
"""

from __future__ import annotations

import subprocess
import sys
import sysconfig
import tempfile
from pathlib import Path

SRC = Path("/root/reference/pkg/src/voltyard/backends/_kernel.pyx")
DEST = Path(__file__).resolve().parent / "_ref"


def build(quiet: bool = True) -> Path | None:
    if not SRC.exists():
        return None
    DEST.mkdir(exist_ok=True)
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    target = DEST / f"_kernel{suffix}"
    if target.exists() and target.stat().st_mtime >= SRC.stat().st_mtime:
        return target
    with tempfile.TemporaryDirectory() as tmp:
        c_file = Path(tmp) / "_kernel.c"
        subprocess.run([sys.executable, "-m", "cython", "-3", "-o", str(c_file), str(SRC)], check=True,
                       capture_output=quiet)
        inc = sysconfig.get_paths()["include"]
        subprocess.run(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", f"-I{inc}", str(c_file),
                        "-o", str(target)], check=True, capture_output=quiet)
    return target


if __name__ == "__main__":
    print(build(quiet=False))
