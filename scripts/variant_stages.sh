#!/bin/bash
# Rebuild libkpme_b200.so with each set of -D flags and print the eager
# per-stage device times (scripts/stage_times.py) for configs 2-4.
# Usage: scripts/variant_stages.sh "FLAGS1" "FLAGS2" ...   (restores the default build)
cd "$(dirname "$0")/.."
for flags in "$@"; do
  make -C paper_2601_18838_b200/csrc clean > /dev/null
  make -C paper_2601_18838_b200/csrc -j8 NVEXTRA="$flags" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  echo "== $flags"
  python scripts/stage_times.py cfg2 cfg3 cfg4 2>/dev/null
done
make -C paper_2601_18838_b200/csrc clean > /dev/null
make -C paper_2601_18838_b200/csrc -j8 > /dev/null 2>&1
