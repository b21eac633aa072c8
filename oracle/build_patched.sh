#!/bin/bash
# Builds the reference WITH the B200 drop-in applied (INTEGRATION.md section
# 2, oracle/patchdb_b200.patch) -- test infrastructure, outputs only under
# oracle/_ref/patched/ (git-ignored; it travels to the GPU box):
#   acceptance                the reference's tests/acceptance.cpp (10 criteria)
#   patchdb/_core*.so         the reference's pybind11 module (bindings/py_module.cpp)
#   patchdb/__init__.py       the reference's python package file, copied as built
#   test_smoke.py             the reference's tests/python/test_smoke.py, copied as built
# and, as the comparison arm, the UNPATCHED pybind11 module under
# oracle/_ref/unpatched/patchdb/ (same flags, no libpdb_cuda.so).
# The patched sources live in a scratch copy under /tmp; /root/reference is
# only read.  Every binary links paper_1812_07607_b200/libpdb_cuda.so.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/.." && pwd)
REF=${PATCHDB_REF:-/root/reference/proj}
JSON_INC=${JSON_INC:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}
OUT=$HERE/_ref/patched
SRC=$(mktemp -d /tmp/pdb_patched.XXXXXX)
trap 'rm -rf "$SRC"' EXIT
cp -r "$REF/." "$SRC/"
chmod -R u+w "$SRC"
(cd "$SRC" && patch -p1 --quiet < "$HERE/patchdb_b200.patch")
mkdir -p "$OUT/patchdb" "$SRC/obj"
# the system g++ (links the shared libstdc++ the Python process and torch use;
# a static libstdc++ copy inside the module breaks once torch is loaded)
CXX=${PDB_PATCHED_CXX:-/usr/bin/g++}
# the reference's own Release flags (CMakeLists.txt:7-9 -> -O3 -DNDEBUG)
FLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -pthread -I$SRC/include -I$JSON_INC -I$ROOT/include"
pids=()
for f in core record_store storage index etl query bench planfile; do
  $CXX $FLAGS -c "$SRC/src/$f.cpp" -o "$SRC/obj/$f.o" & pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
ar rcs "$SRC/obj/libpatchdb_core.a" "$SRC"/obj/*.o
LIBDIR=$ROOT/paper_1812_07607_b200
$CXX $FLAGS -I"$SRC/tests" -o "$OUT/acceptance" "$SRC/tests/acceptance.cpp" \
    "$SRC/obj/libpatchdb_core.a" -L"$LIBDIR" -l:libpdb_cuda.so \
    -Wl,-rpath,'$ORIGIN/../../../paper_1812_07607_b200' -lz
PYINC=$(python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PBINC=$(python3 -c "import pybind11; print(pybind11.get_include())")
EXT=$(python3 -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
$CXX $FLAGS -shared -fvisibility=hidden -I"$PYINC" -I"$PBINC" -o "$OUT/patchdb/_core$EXT" \
    "$SRC/bindings/py_module.cpp" "$SRC/obj/libpatchdb_core.a" -L"$LIBDIR" -l:libpdb_cuda.so \
    -Wl,-rpath,'$ORIGIN/../../../../paper_1812_07607_b200' -lz
cp "$SRC/python/patchdb/__init__.py" "$OUT/patchdb/__init__.py"
# the unpatched module: the same sources before the patch
UN=$HERE/_ref/unpatched
mkdir -p "$UN/patchdb" "$SRC/orig/obj"
cp -r "$REF/." "$SRC/orig/"
chmod -R u+w "$SRC/orig"
UFLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -pthread -I$SRC/orig/include -I$JSON_INC"
pids=()
for f in core record_store storage index etl query bench planfile; do
  $CXX $UFLAGS -c "$SRC/orig/src/$f.cpp" -o "$SRC/orig/obj/$f.o" & pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
$CXX $UFLAGS -shared -fvisibility=hidden -I"$PYINC" -I"$PBINC" -o "$UN/patchdb/_core$EXT" \
    "$SRC/orig/bindings/py_module.cpp" "$SRC"/orig/obj/*.o -lz
cp "$SRC/orig/python/patchdb/__init__.py" "$UN/patchdb/__init__.py"
cp "$SRC/tests/python/test_smoke.py" "$OUT/test_smoke.py"
echo "patched reference built into $OUT"
