#!/bin/bash
# On the GPU box: the default bench line, the ncu launch list of the device
# path and of a short bench run, and ncu --set full captures of the pipeline
# kernels (config 3) and of the config-5 DGEMM. Each ncu command runs only
# after the same command exited 0 without ncu. Outputs in gpurun_out/; the
# summaries are copied into profiles/ afterwards.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || { tail -20 gpurun_out/bench.err; exit 1; }
cat gpurun_out/bench.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_step.py cfg3 3 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv \
    python scripts/profile_step.py cfg3 3 > gpurun_out/ncu_launch_step.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_spread|k_bwd_gather|k_gather_cc|k_col_scatter|k_z_sort|k_tile_hist|k_col_scan|k_tile_sort|k_tile_keys|k_z_tiles|k_core_sum" -c 5 \
    -f -o gpurun_out/full python scripts/profile_step.py cfg3 1 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
python scripts/dense_once.py 256 16 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_dgemm" -c 3 \
    -f -o gpurun_out/full_dgemm python scripts/dense_once.py 256 16 > gpurun_out/ncu_dgemm.log 2>&1
tail -1 gpurun_out/ncu_dgemm.log
