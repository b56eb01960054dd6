"""Build the native library in-tree: paper_2512_09472_b200/_lib/libwarmserve.so.

nvcc cross-compiles every CUDA source for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's
source page maps to the code. The CUDA runtime is linked statically and the
driver API is resolved at run time, so the library loads on GPU-less hosts
(ledger-only pools) and on the B200 box alike.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libwarmserve.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
          f"-I{INCLUDE}", f"-I{CSRC}"]
CUDA_ONLY = ["--expt-relaxed-constexpr", "-Xptxas", "-O3"]
if os.environ.get("WS_DEBUG_WAIT"):  # watchdog build of the mbarrier waits (debugging only)
    CUDA_ONLY.append("-DWS_DEBUG_WAIT")
if os.environ.get("WS_ATTN_TRACE"):  # clock64 timeline of one attention CTA (debugging only)
    CUDA_ONLY.append("-DWS_ATTN_TRACE")
if os.environ.get("WS_ATTN_POLY"):  # pairs of every 8 whose exp2 runs on the FMA-pipe polynomial (A/B builds)
    CUDA_ONLY.append(f"-DWS_ATTN_POLY={int(os.environ['WS_ATTN_POLY'])}")
if os.environ.get("WS_ATTN_SPLIT"):  # 0: one softmax warp per 32 query rows of a tile (A/B builds)
    CUDA_ONLY.append(f"-DWS_ATTN_SPLIT={int(os.environ['WS_ATTN_SPLIT'])}")
if os.environ.get("WS_DEC_KVPOL"):  # decode-attention K/V L2 policy: 1 evict_first, 2 evict_last (A/B builds)
    CUDA_ONLY.append(f"-DWS_DEC_KVPOL={int(os.environ['WS_DEC_KVPOL'])}")
if os.environ.get("WS_DEC_STAGES"):  # decode-attention ring depth per warp (A/B builds)
    CUDA_ONLY.append(f"-DWS_DEC_STAGES={int(os.environ['WS_DEC_STAGES'])}")
if os.environ.get("WS_SKINNY_TRACE"):  # per-CTA globaltimer timeline of the skinny GEMM (debugging only)
    CUDA_ONLY.append("-DWS_SKINNY_TRACE")
if os.environ.get("WS_GEMM_TRACE"):  # per-CTA globaltimer timeline of the pair GEMM (debugging only)
    CUDA_ONLY.append("-DWS_GEMM_TRACE")


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(p for p in CSRC.rglob("*") if p.suffix in (".cu", ".cpp"))


def _headers():
    return [p for p in CSRC.rglob("*") if p.suffix in (".h", ".cuh")] + list(INCLUDE.glob("*.h"))


def _compile(src: Path, obj: Path, verbose: bool) -> str:
    cmd = [_nvcc(), *ARCH, *COMMON]
    if src.suffix == ".cu":
        cmd += CUDA_ONLY
        if os.environ.get("WS_PTXAS_V"):
            cmd += ["-Xptxas", "-v"]
    cmd += ["-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False, force: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    obj_dir = OUT_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)
    newest_header = max((p.stat().st_mtime for p in _headers()), default=0.0)
    jobs = []
    objs = []
    for src in _sources():
        obj = obj_dir / (src.relative_to(CSRC).as_posix().replace("/", "_") + ".o")
        objs.append(obj)
        stale = force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_header)
        if stale:
            jobs.append((src, obj))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        futs = {ex.submit(_compile, s, o, verbose): s for s, o in jobs}
        for f in cf.as_completed(futs):
            log = f.result()
            if log.strip() and (verbose or os.environ.get("WS_PTXAS_V")):
                print(f"[{futs[f].name}]\n{log}", file=sys.stderr)
    if jobs or force or not LIB.exists():
        cmd = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
               "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
