#!/bin/sh
# Protocol-check build (race evidence while compute-sanitizer is closed on this
# pool): libgg_checked.so with -DGG_CHECK_PROTOCOLS, whose kernels __trap() if a
# warp-private stamp ranking disagrees with __match_any_sync, a depth block is
# not stably sorted after staging, or a tile-list slot is written twice.
# Run the GPU tests against it with GG_LIB=paper_2510_15352_b200/libgg_checked.so.
HERE="$(cd "$(dirname "$0")" && pwd)"
EXTRA="-DGG_CHECK_PROTOCOLS" BUILD_DIR="$HERE/build_checked" LIB="$HERE/libgg_checked.so" sh "$HERE/build.sh"
