#!/bin/bash
# Builds build/integrated_api: the reference patched per INTEGRATION.md §1-3
# (a scratch copy outside this repository, tests/native/integrate_reference.py),
# compiled in its own namespace together with the adapter and linked with
# libfvb.so.  Objects only land in build/integrated/.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${REF:-/root/reference/proj}"
CUDA="${CUDA:-/usr/local/cuda}"
SCRATCH="$(mktemp -d /tmp/fvb_integrated.XXXXXX)"
trap 'rm -rf "$SCRATCH"' EXIT
python3 "$HERE/integrate_reference.py" "$REF" "$SCRATCH"
OUT="$HERE/build/integrated"
mkdir -p "$OUT"
CXXFLAGS="-std=c++20 -O3 -DNDEBUG -ffp-contract=off -fPIC -pthread -I$SCRATCH/include -I$ROOT/include \
  -I$ROOT/paper_1809_09851_b200/host -I$CUDA/include"
OBJS=()
PIDS=()
for f in "$SCRATCH"/src/*.cpp "$ROOT/paper_1809_09851_b200/host/fusevec_device.cpp" \
         "$ROOT/paper_1809_09851_b200/host/fusevec_device_bench.cpp"; do
  o="$OUT/$(basename "${f%.cpp}").o"
  g++ $CXXFLAGS -I"$SCRATCH/src" -c "$f" -o "$o" &
  PIDS+=($!)
  OBJS+=("$o")
done
for p in "${PIDS[@]}"; do wait "$p"; done  # set -e: any failed compile stops the build
g++ $CXXFLAGS -Wall -o "$HERE/build/integrated_api" "$HERE/integrated_api.cpp" "${OBJS[@]}" \
  -L"$ROOT/paper_1809_09851_b200/lib" -lfvb -L"$CUDA/lib64" -lcudart \
  -Wl,-rpath,'$ORIGIN/../../../paper_1809_09851_b200/lib' -Wl,-rpath,"$CUDA/lib64" -ldl -pthread
echo "built $HERE/build/integrated_api"

# The reference's own unit tests (proj/tests/test_*.cpp, compiled where they
# lie, with the doctest stand-in of doctest_shim/) against a second build of
# the integrated reference whose Backend::scalar_ref() can be switched to the
# device at run time (FUSEVEC_SCALAR_REF_IS_DEVICE).
SCRATCH2="$(mktemp -d /tmp/fvb_integrated_sw.XXXXXX)"
trap 'rm -rf "$SCRATCH" "$SCRATCH2"' EXIT
python3 "$HERE/integrate_reference.py" "$REF" "$SCRATCH2" --scalar-ref-switch
OUT2="$HERE/build/integrated_sw"
mkdir -p "$OUT2"
CXX2="-std=c++20 -O2 -DNDEBUG -ffp-contract=off -fPIC -pthread -I$SCRATCH2/include -I$ROOT/include \
  -I$ROOT/paper_1809_09851_b200/host -I$CUDA/include"
OBJS2=()
PIDS=()
for f in "$SCRATCH2"/src/*.cpp "$ROOT/paper_1809_09851_b200/host/fusevec_device.cpp" \
         "$ROOT/paper_1809_09851_b200/host/fusevec_device_bench.cpp"; do
  o="$OUT2/$(basename "${f%.cpp}").o"
  g++ $CXX2 -I"$SCRATCH2/src" -c "$f" -o "$o" &
  PIDS+=($!)
  OBJS2+=("$o")
done
for f in "$REF"/tests/doctest_main.cpp "$REF"/tests/test_*.cpp; do
  o="$OUT2/t_$(basename "${f%.cpp}").o"
  g++ $CXX2 -I"$HERE/doctest_shim" -I"$REF/tests" -c "$f" -o "$o" &
  PIDS+=($!)
  OBJS2+=("$o")
done
for p in "${PIDS[@]}"; do wait "$p"; done
# and the reference's acceptance criteria (proj/tests/acceptance.cpp) on the same build
g++ $CXX2 -I"$REF/tests" -DFUSEVEC_TEST_DIR="\"$REF/tests\"" -c "$REF/tests/acceptance.cpp" \
  -o "$OUT2/acceptance.o"
LIBOBJS=()
for o in "${OBJS2[@]}"; do case "$o" in */t_*) ;; *) LIBOBJS+=("$o");; esac; done
g++ -pthread -o "$HERE/build/reference_acceptance" "$OUT2/acceptance.o" "${LIBOBJS[@]}" \
  -L"$ROOT/paper_1809_09851_b200/lib" -lfvb -L"$CUDA/lib64" -lcudart \
  -Wl,-rpath,'$ORIGIN/../../../paper_1809_09851_b200/lib' -Wl,-rpath,"$CUDA/lib64" -ldl
g++ -pthread -o "$HERE/build/reference_unit_tests" "${OBJS2[@]}" \
  -L"$ROOT/paper_1809_09851_b200/lib" -lfvb -L"$CUDA/lib64" -lcudart \
  -Wl,-rpath,'$ORIGIN/../../../paper_1809_09851_b200/lib' -Wl,-rpath,"$CUDA/lib64" -ldl
echo "built $HERE/build/reference_unit_tests"

