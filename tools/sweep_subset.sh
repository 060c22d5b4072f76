#!/bin/bash
# time a subset of configs: tools/sweep_subset.sh C3-Q1 C3-Q2 ...
cd "$(dirname "$0")/.."
for c in "$@"; do
  python tools/profile_apply.py --config $c --time --reps 20 2>/dev/null | tail -1 || echo "{\"config\": \"$c\", \"error\": true}"
done
