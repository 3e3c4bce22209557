#!/bin/sh
# Builds libgg.so (the CUDA product path) for sm_100a, in-tree.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
NVCC="${NVCC:-nvcc}"
OUT="$HERE/build"
mkdir -p "$OUT"
FLAGS="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I$ROOT/include -Xptxas -v"
pids=""
for f in "$HERE"/csrc/*.cu; do
  b=$(basename "$f" .cu)
  $NVCC $FLAGS -c "$f" -o "$OUT/$b.o" > "$OUT/$b.ptxas.log" 2>&1 || { cat "$OUT/$b.ptxas.log"; exit 1; } &
  pids="$pids $!"
done
fail=0
for p in $pids; do wait $p || fail=1; done
[ $fail -eq 0 ] || exit 1
$NVCC -shared -gencode arch=compute_100a,code=sm_100a -o "$HERE/libgg.so" "$OUT"/*.o
echo "built $HERE/libgg.so"
