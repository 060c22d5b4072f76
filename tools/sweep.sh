#!/bin/bash
# Time every BASELINE config on one GPU (CUDA events, L2 flushed between
# applies) -> one JSON line per config.
cd "$(dirname "$0")/.."
for c in C1 C2-P1 C2-P2 C2-P3 C2-P4 C3-Q1 C3-Q2 C3-Q3 C3-Q4 C3-Q5 C3-Q6 \
         C4-quad-Q1 C4-quad-Q2 C4-quad-Q3 C4-quad-Q4 C4-hex-Q1 C4-hex-Q2 C4-hex-Q3 C5 C6; do
  python tools/profile_apply.py --config $c --time --reps 20 2>/dev/null || echo "{\"config\": \"$c\", \"error\": true}"
done
