"""Build libbluefog_b200.so in-tree (sm_100a only).

    python -m paper_2111_04287_b200.build

nvcc cross-compiles without a GPU.  The .so is git-ignored but travels to the
GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libbluefog_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(HERE, "..", "include", "bluefog_b200.h"))
    return os.path.getmtime(SO) >= max(os.path.getmtime(p) for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = SO) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file),
    then link the shared library.  defines: extra -D flags for tuning variants."""
    if not force and out == SO and not defines and up_to_date():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    import tempfile

    obj_dir = tempfile.mkdtemp(prefix="bf_build_")
    compile_flags = [f for f in FLAGS if f != "-shared"]
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [NVCC, *compile_flags, *dflags, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, res

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    log_text = ""
    failed = False
    for src, obj, cmd, res in results:
        log_text += " ".join(cmd) + "\n" + res.stdout + res.stderr
        failed |= res.returncode != 0
    if not failed:
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               *[obj for _, obj, _, _ in results], "-o", out + ".tmp"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log_text += " ".join(cmd) + "\n" + res.stdout + res.stderr
        failed = res.returncode != 0
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(log_text)
    for _, obj, _, _ in results:
        if os.path.exists(obj):
            os.unlink(obj)
    os.rmdir(obj_dir)
    if failed:
        sys.stderr.write(log_text[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(out + ".tmp", out)
    if verbose:
        sys.stdout.write(log_text)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else SO))
