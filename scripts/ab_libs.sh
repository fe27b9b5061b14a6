#!/bin/bash
# A/B of library variants (paper_2207_05495_b200/lib_ab/*.so) against the main build on
# the engine-only solve time (scripts/ab_solve.py).  Usage: scripts/ab_libs.sh [spec:R ...]
cd "$(dirname "$0")/.."
for lib in paper_2207_05495_b200/lib/libsynchro_b200.so paper_2207_05495_b200/lib_ab/*.so; do
  echo "== $lib"
  SYNCHRO_B200_LIB=$PWD/$lib python scripts/ab_solve.py "$@"
done
