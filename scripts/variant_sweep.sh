#!/bin/bash
# Rebuild libkpme_b200.so with each set of -D flags and record per-kernel
# times (ncu launch list) for config 3. Usage: scripts/variant_sweep.sh "FLAGS1" "FLAGS2" ...
# Restores the default build at the end.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for flags in "$@"; do
  make -C paper_2601_18838_b200/csrc clean > /dev/null
  make -C paper_2601_18838_b200/csrc -j8 NVEXTRA="$flags" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  PROFILE_NOCHECK=1 python scripts/profile_step.py cfg3 3 > /dev/null 2>&1 || { echo "run failed: $flags"; continue; }
  tag=$(echo "$flags" | tr -c 'A-Za-z0-9' '_')
  PROFILE_NOCHECK=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/var_$tag.csv \
      python scripts/profile_step.py cfg3 3 > /dev/null 2>&1
  echo "== $flags"
  python scripts/launches.py gpurun_out/var_$tag.csv | grep -E "${SWEEP_GREP:-spread|gather|keys|place|segsort}"
done
make -C paper_2601_18838_b200/csrc clean > /dev/null
make -C paper_2601_18838_b200/csrc -j8 > /dev/null 2>&1
