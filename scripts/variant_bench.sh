#!/bin/bash
# Rebuild libkpme_b200.so with each set of -D flags and print the bench's
# graph-replayed ms/step and eager per-stage times for config 3 (the numbers
# the bench line reports; ncu launch lists replay kernels cold).
# Usage: scripts/variant_bench.sh "FLAGS1" "FLAGS2" ...   (restores the default build)
cd "$(dirname "$0")/.."
for flags in "$@"; do
  make -C paper_2601_18838_b200/csrc clean > /dev/null
  make -C paper_2601_18838_b200/csrc -j8 NVEXTRA="$flags" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  echo "== $flags"
  python bench.py --no-cpu-baseline --no-extras --steps 30 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('  ms/step %.4f  e2e %.4f  stages %s' % (d['ms_per_step'], d['e2e']['ms_per_step'],
      {k: round(v * 1e3, 1) for k, v in d['stages'].items()}))"
done
make -C paper_2601_18838_b200/csrc clean > /dev/null
make -C paper_2601_18838_b200/csrc -j8 > /dev/null 2>&1
