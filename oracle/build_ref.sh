#!/usr/bin/env bash
# Build the UNMODIFIED reference package (gvplan, /root/reference/pkg) into
# oracle/_ref/ so it can be imported as the CPU checker and timed as the
# `--impl reference` arm. Test infrastructure only: nothing under oracle/ is
# on the product path.
#
# The reference's own build is setup.py + Cython (pkg/setup.py:1-26). We build
# from a scratch copy under /tmp (the reference tree is read-only) with the
# system gcc (the /opt gcc lacks libgomp.spec), then copy the
# built package (Python sources + the compiled _kernels extension) into
# oracle/_ref/gvplan. oracle/_ref is git-ignored and travels to the GPU box.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${GVPLAN_REFERENCE:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: reference not present at $REF; keeping existing $OUT" >&2
  exit 0
fi
SCRATCH="$(mktemp -d /tmp/gvplan_ref.XXXXXX)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$REF"/. "$SCRATCH"/
cd "$SCRATCH"
PY="${PYTHON:-python3}"
CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" "$PY" setup.py build_ext --inplace >"$SCRATCH/build.log" 2>&1 || {
  echo "build_ref: OpenMP build failed, retrying with GVPLAN_NO_OPENMP=1" >&2
  GVPLAN_NO_OPENMP=1 CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" "$PY" setup.py build_ext --inplace >>"$SCRATCH/build.log" 2>&1
}
rm -rf "$OUT"
mkdir -p "$OUT"
cp -r "$SCRATCH/src/gvplan" "$OUT/gvplan"
rm -rf "$OUT/gvplan/__pycache__" "$OUT/gvplan"/*.c "$OUT/gvplan"/*.pyx
# the reference's own test suite, unmodified, so tools/run_reference_suite.py
# can run it against paper_2411_03416_b200 on the GPU box (git-ignored like
# the rest of oracle/_ref)
cp -r "$REF/tests" "$OUT/tests"
rm -rf "$OUT/tests/__pycache__"
echo "built reference into $OUT:"
ls "$OUT/gvplan" "$OUT/tests"
