#!/usr/bin/env bash
# Profiling evidence for profiles/ (run under gpurun on ONE GPU; gpurun_out/ must stay < 64 MiB,
# so the captures are split: PART=1 launch list + Legendre capture + bench lines, PART=2 the
# ring-stage captures).
set -u
mkdir -p gpurun_out
if [ "${PART:-1}" = "1" ]; then
  # launch list of the bench command (cold-cache, serialised: shares, not absolutes)
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  # one full capture of each C4 Legendre kernel
  ncu --set full --clock-control none --import-source on -k regex:"leg_alm2map_kernel|leg_map2alm_kernel" -c 2 \
      -o gpurun_out/c4_legendre python tools/profile_run.py --nside 2048 --lmax 4096 > /dev/null 2>&1
  python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
else
  # ring stage: the power-of-two engine's synthesis classes (Bluestein 8192..256, belt direct 4096)
  # and the analysis ones (launches 11..17)
  ncu --set full --clock-control none -k regex:"ring_p2" -c 7 \
      -o gpurun_out/c4_ring_synth python tools/profile_run.py --nside 2048 --lmax 4096 > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:"ring_p2" --launch-skip 11 -c 7 \
      -o gpurun_out/c4_ring_anal python tools/profile_run.py --nside 2048 --lmax 4096 > /dev/null 2>&1
fi
du -sh gpurun_out
