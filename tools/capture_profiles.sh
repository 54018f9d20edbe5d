#!/usr/bin/env bash
# Profiling evidence for profiles/ (run under gpurun on ONE GPU).
set -u
mkdir -p gpurun_out
# launch list of the bench command (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# one full capture of each C4 Legendre kernel and every ring-FFT class
ncu --set full --clock-control none --import-source on -k regex:"leg_alm2map_kernel|leg_map2alm_kernel" -c 2 \
    -o gpurun_out/c4_legendre python tools/profile_run.py --nside 2048 --lmax 4096 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ring_" -c 8 \
    -o gpurun_out/c4_ring python tools/profile_run.py --nside 2048 --lmax 4096 > /dev/null 2>&1
ls -la gpurun_out
