#!/bin/sh
# Builds libgg.so (the CUDA product path) for sm_100a, in-tree.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
NVCC="${NVCC:-nvcc}"
OUT="${BUILD_DIR:-$HERE/build}"
LIB="${LIB:-$HERE/libgg.so}"
mkdir -p "$OUT"
FLAGS="$EXTRA -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I$ROOT/include -Xptxas -v"
pids=""
for f in "$HERE"/csrc/*.cu; do
  b=$(basename "$f" .cu)
  $NVCC $FLAGS -c "$f" -o "$OUT/$b.o" > "$OUT/$b.ptxas.log" 2>&1 || { cat "$OUT/$b.ptxas.log"; exit 1; } &
  pids="$pids $!"
done
fail=0
for p in $pids; do wait $p || fail=1; done
[ $fail -eq 0 ] || exit 1
$NVCC -shared -gencode arch=compute_100a,code=sm_100a -o "$LIB" "$OUT"/*.o
echo "built $LIB"
