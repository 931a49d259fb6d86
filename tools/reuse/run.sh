#!/bin/bash
# Pair-reuse analysis of the reference build on a C-config prefix (CPU, oracle):
# how many of scan_vertex's pair checks repeat a pair evaluated earlier in
# the same build (exact set), and the hit rate of direct-mapped memo tables.
# usage: tools/reuse/run.sh ROWS CFG DIM LOG2_SMALLEST_TABLE   (e.g. 50000 3 960 18)
set -e
HERE=$(cd "$(dirname "$0")" && pwd); ROOT=$(cd "$HERE/../.." && pwd); T=$(mktemp -d)
# the oracle's scan_vertex with its l2_sq call routed through the counting hook
sed 's/float dvw = ro_l2_sq(data + (uint64_t)v.id \* d, data + (uint64_t)w->id \* d, d);/float dvw = hook_l2(v.id, w->id, data, d);/' \
  "$ROOT/oracle/rnnd_oracle.c" > "$T/oracle_hooked.c"
grep -q hook_l2 "$T/oracle_hooked.c"
cp "$HERE/pair_reuse.c" "$T/"
g++ -O3 -march=native -ffp-contract=off -x c "$T/pair_reuse.c" -x c++ "$ROOT/datagen/datagen.cpp" \
  -I"$ROOT/oracle" -I"$T" -o "$T/pair_reuse"
"$T/pair_reuse" "$@"
