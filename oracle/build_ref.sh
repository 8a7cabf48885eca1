#!/usr/bin/env bash
# Build the reference's own compiled stride kernel into oracle/_ref/.
#
# TEST INFRASTRUCTURE: the output is the CPU reference that tests and
# bench.py (--impl reference, cpu_baseline) time and check against.  The
# reference source is read in place from /root/reference (read-only); only
# generated C and the built extension land in oracle/_ref/ (git-ignored).
#
# Flags are the reference's own (pkg/setup.py:43-50): -O3 -fopenmp
# -ffp-contract=off.  System gcc is used explicitly (an
# /opt/gcc without libgomp.spec silently drops OpenMP).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${SVSIM_REF:-/root/reference}/pkg/src/svsim/kernel/_stride_cy.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
    echo "build_ref: reference source $SRC not present; skipping" >&2
    exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python3}"
EXT="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
INC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
"$PY" -m cython -3 -o "$OUT/_stride_cy.c" "$SRC"
/usr/bin/gcc -O3 -fopenmp -ffp-contract=off -fPIC -shared -I"$INC" \
    "$OUT/_stride_cy.c" -o "$OUT/_stride_cy$EXT"
echo "build_ref: built $OUT/_stride_cy$EXT"
# the reference's pure-Python package + kernel tests, with INTEGRATION.md's
# cuda-backend registration applied (tests/test_gpu_plug.py runs them)
"$PY" "$HERE/stage_ref_pkg.py" "${SVSIM_REF:-/root/reference}"
