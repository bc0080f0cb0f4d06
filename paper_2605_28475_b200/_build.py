"""In-tree build of ``libbfq.so`` for sm_100a, with source provenance.

Every translation unit compiles in parallel into ``build/obj/`` (an object is
reused only when the hash of its source, every header and the flags is
unchanged).  The link step adds a generated unit carrying the hash of the whole
source tree (``bfq_build_id()``, and the marker string ``BFQ_BUILD_ID=<hash>``
in the binary), so the loader (``_lib.py``) can refuse -- or rebuild -- a
library that was not compiled from the sources next to it.

``checked=True`` (or ``"checked"``) builds ``libbfq_checked.so``: the same
sources with ``-DBFQ_CHECKED`` (device-side bounds checks on every
shared-memory and table access, mbarrier wait timeouts, R-ring / Phi
poisoning), for the self-checking GPU tests (tests/test_gpu_checked.py).
``"timing"`` builds ``libbfq_timing.so`` with ``-DBFQ_PHASE_CLOCKS``: per-phase
cycle counters and the BFQ_DEBUG stage-skip switches of the timing
experiments (results are wrong in the skip modes; never used by tests).
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v"]
SOURCES = [
    "bfq_cuda.cu", "bfq_plan.cpp", "bfr_build.cu", "bfq_project.cu", "bfq_project_samples.cu",
    "bfq_inst_n5.cu", "bfq_inst_n9.cu", "bfq_inst_n11.cu", "bfq_inst_n13.cu", "bfq_inst_n17.cu",
    "bfq_inst_generic.cu",
]
HEADER_EXT = (".h", ".cuh", ".hpp")


VARIANTS = {"": [], "checked": ["-DBFQ_CHECKED=1"], "timing": ["-DBFQ_PHASE_CLOCKS=1"],
            # A/B experiments: the timing build plus -DBFQ_EXPERIMENT (kernel code paths under test)
            "exp": ["-DBFQ_PHASE_CLOCKS=1", "-DBFQ_EXPERIMENT=1"]}


def _variant(checked) -> str:
    """True / False (the checked build or not) or a variant name."""
    if checked is True:
        return "checked"
    if not checked:
        return ""
    if checked not in VARIANTS:
        raise ValueError(f"unknown library variant {checked!r}")
    return checked


def lib_path(checked=False) -> str:
    v = _variant(checked)
    return os.path.join(PKG, f"libbfq_{v}.so" if v else "libbfq.so")


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(HEADER_EXT)]
    hs += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(HEADER_EXT)]
    return sorted(hs)


def _digest(paths, extra: str) -> str:
    h = hashlib.sha256(extra.encode())
    for p in paths:
        h.update(os.path.relpath(p, ROOT).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:24]


def _defines(checked) -> list[str]:
    return VARIANTS[_variant(checked)]


def source_hash(checked=False) -> str:
    """Hash of every source, header and flag the library is built from."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    return _digest(srcs + _headers(), " ".join(NVCC_FLAGS + _defines(checked) + SOURCES))


def embedded_hash(path: str) -> str | None:
    """The BFQ_BUILD_ID marker of a built library, or None."""
    try:
        with open(path, "rb") as fh:
            blob = fh.read()
    except OSError:
        return None
    i = blob.find(b"BFQ_BUILD_ID=")
    if i < 0:
        return None
    j = i + len(b"BFQ_BUILD_ID=")
    return blob[j:j + 24].decode(errors="replace")


def is_current(checked=False) -> bool:
    return embedded_hash(lib_path(checked)) == source_hash(checked)


def build(checked=False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile (only what changed) and link; returns the library path."""
    path = lib_path(checked)
    want = source_hash(checked)
    if embedded_hash(path) == want:
        if verbose:
            print(f"{os.path.basename(path)} up to date ({want})")
        return path
    os.makedirs(BUILD, exist_ok=True)
    hdr_hash = _digest(_headers(), " ".join(NVCC_FLAGS + _defines(checked)))
    tag = {"": "opt", "checked": "chk", "timing": "tim", "exp": "exp"}[_variant(checked)]

    def compile_one(src):
        full = os.path.join(CSRC, src)
        oh = _digest([full], hdr_hash)
        obj = os.path.join(BUILD, f"{src}.{tag}.{oh}.o")
        if os.path.exists(obj):
            return obj, ""
        cmd = [NVCC, *NVCC_FLAGS, *_defines(checked), "-I", INCLUDE, "-I", CSRC, "-c", full, "-o", obj + ".tmp"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}{res.stderr}")
        os.replace(obj + ".tmp", obj)
        return obj, res.stderr

    jobs = jobs or max(1, min(len(SOURCES), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose:
        for _, log in results:
            sys.stdout.write(log)
    idsrc = os.path.join(BUILD, f"build_id.{tag}.{want}.cpp")
    with open(idsrc, "w") as fh:
        fh.write('// generated by _build.py: provenance of this library\n'
                 f'static const char kId[] = "BFQ_BUILD_ID={want}";\n'
                 'extern "C" const char* bfq_build_id(void) { return kId + 13; }\n')
    idobj = idsrc[:-4] + ".o"
    res = subprocess.run(["g++", "-O2", "-fPIC", "-c", idsrc, "-o", idobj], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("g++ failed on the build-id unit:\n" + res.stderr)
    tmp = path + ".tmp"
    res = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *[o for o, _ in results], idobj],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link of {os.path.basename(path)} failed:\n{res.stdout}{res.stderr}")
    os.replace(tmp, path)
    if verbose:
        print(f"built {path} ({want})")
    return path
