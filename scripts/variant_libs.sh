#!/bin/bash
# Eager per-stage device times (scripts/stage_times.py) for prebuilt variant libraries
# (scripts/build_variant.sh). Usage: scripts/variant_libs.sh "cfg3 cfg4" tag1 tag2 ...
cd "$(dirname "$0")/.."
cfgs=$1; shift
for tag in "$@"; do
  lib=paper_2601_18838_b200/variants/libkpme_$tag.so
  [ "$tag" = default ] && lib=paper_2601_18838_b200/libkpme_b200.so
  echo "== $tag $(PROFILE_NOCHECK=1 KPME_LIB=$PWD/$lib python scripts/stage_times.py $cfgs 2>&1 | tail -n 1)"
done
