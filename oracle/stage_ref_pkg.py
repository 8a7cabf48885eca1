"""Stage the reference's pure-Python package and its kernel tests into
oracle/_ref/pkg (git-ignored; travels to the GPU box with the snapshot) and
apply INTEGRATION.md section 1's registration of the ``cuda`` backend to the
staged copy of ``svsim/kernel/__init__.py``.

TEST INFRASTRUCTURE ONLY: tests/test_gpu_plug.py runs the reference's own
``pkg/tests/test_kernel.py`` against this staged package so the plug-in seam
(kernel/__init__.py:62-75) is exercised by the reference's tests, not by ours.
The product package never imports anything staged here.  /root/reference is
read in place and never written.

usage: python oracle/stage_ref_pkg.py [REFERENCE_ROOT]
"""

from __future__ import annotations

import glob
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "pkg")

# INTEGRATION.md section 1, applied verbatim to the staged kernel/__init__.py.
# Each (anchor, replacement) must match exactly once, or staging fails loudly.
PATCH = [
    (
        'BACKEND = "compiled" if _stride_cy is not None else "python"\n',
        "try:\n"
        "    from paper_1801_01037_b200 import backend as _stride_cuda   # B200 engine\n"
        "except Exception:                                              # no GPU / not built\n"
        "    _stride_cuda = None\n"
        "\n"
        'BACKEND = "compiled" if _stride_cy is not None else "python"\n',
    ),
    (
        'def available_backends() -> tuple[str, ...]:\n'
        '    return ("python", "compiled") if _stride_cy is not None else ("python",)\n',
        'def available_backends() -> tuple[str, ...]:\n'
        '    names = ("python", "compiled") if _stride_cy is not None else ("python",)\n'
        '    return names + (("cuda",) if _stride_cuda is not None else ())\n',
    ),
    (
        '    raise ValidationError(f"unknown kernel backend {backend!r}")\n',
        '    if backend == "cuda":\n'
        '        if _stride_cuda is None:\n'
        '            raise ValidationError("cuda kernel is not available in this build")\n'
        '        return _stride_cuda\n'
        '    raise ValidationError(f"unknown kernel backend {backend!r}")\n',
    ),
]


def stage(ref_root: str) -> None:
    src_pkg = os.path.join(ref_root, "pkg", "src", "svsim")
    src_tests = os.path.join(ref_root, "pkg", "tests")
    if not os.path.isdir(src_pkg):
        print(f"stage_ref_pkg: {src_pkg} not present; skipping", file=sys.stderr)
        return
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    dst_pkg = os.path.join(OUT, "svsim")
    shutil.copytree(src_pkg, dst_pkg, ignore=shutil.ignore_patterns("__pycache__", "*.so", "*.c"))
    # the compiled backend = the reference kernel build_ref.sh just made
    for so in glob.glob(os.path.join(HERE, "_ref", "_stride_cy*.so")):
        shutil.copy2(so, os.path.join(dst_pkg, "kernel", os.path.basename(so)))
    os.makedirs(os.path.join(OUT, "tests"))
    for name in ("conftest.py", "test_kernel.py", "test_engine.py"):
        shutil.copy2(os.path.join(src_tests, name), os.path.join(OUT, "tests", name))
    init = os.path.join(dst_pkg, "kernel", "__init__.py")
    with open(init) as f:
        text = f.read()
    for anchor, repl in PATCH:
        if text.count(anchor) != 1:
            raise SystemExit(f"stage_ref_pkg: patch anchor not found exactly once in {init}:\n{anchor}")
        text = text.replace(anchor, repl)
    with open(init, "w") as f:
        f.write(text)
    print(f"stage_ref_pkg: staged svsim + kernel tests into {OUT} (cuda backend registered)")


if __name__ == "__main__":
    stage(sys.argv[1] if len(sys.argv) > 1 else os.environ.get("SVSIM_REF", "/root/reference"))
