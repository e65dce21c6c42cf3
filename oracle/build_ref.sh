#!/usr/bin/env bash
# Test infrastructure only: compiles the reference's own compiled stepping core
# (/root/reference/pkg/src/perchsim/_accel/_core.pyx, Cython + OpenMP, FP64) into
# oracle/_ref/ so it can serve as the parity checker and the CPU baseline arm of
# bench.py.  Sources are read in place from /root/reference (never copied into the
# repo); every output (generated C, object, .so) lands in oracle/_ref/, which is
# git-ignored and travels to the GPU box with the gpurun snapshot.
#
# The reference's own build (pkg/setup.py:17-29) is NOT run; this recipe mirrors its
# flags (-O3 -fopenmp) with the system gcc (the /opt/gcc wrapper lacks libgomp.spec).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${REF_ROOT:-/root/reference}/pkg/src/perchsim/_accel/_core.pyx"
OUT="$HERE/_ref"
mkdir -p "$OUT"
if [ ! -f "$SRC" ]; then
  echo "build_ref: $SRC not present (GPU box?) - keeping prebuilt oracle/_ref" >&2
  exit 0
fi
PY="${PYTHON:-python}"
EXT_SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
NPINC="$($PY -c 'import numpy; print(numpy.get_include())')"
cython -3 "$SRC" -o "$OUT/_core.c"
/usr/bin/gcc -O3 -fopenmp -fPIC -shared -I"$PYINC" -I"$NPINC" \
  -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  "$OUT/_core.c" -o "$OUT/_core$EXT_SUFFIX" -lgomp
echo "built $OUT/_core$EXT_SUFFIX"
# Stage the unmodified reference package (pure Python + numpy) under oracle/_ref/pkg
# so the drop-in test (tests/test_gpu_dropin.py) can run the reference's own
# mppi.optimize / policy.build_policy / Engine / nmpc.control_loop on the GPU box
# with the CUDA stepping module installed as its _accel._core.  Git-ignored (never
# in history); travels with the gpurun snapshot like the compiled core.
rm -rf "$OUT/pkg"
mkdir -p "$OUT/pkg"
cp -r "${REF_ROOT:-/root/reference}/pkg/src/perchsim" "$OUT/pkg/perchsim"
find "$OUT/pkg" -name __pycache__ -prune -exec rm -rf {} +
chmod -R u+w "$OUT/pkg"
echo "staged $OUT/pkg/perchsim"
