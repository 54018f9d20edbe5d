set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
for f in fp64_probe fp64_mix_probe leg_pattern_probe; do timeout 120 ./tools/$f.bin > gpurun_out/$f.txt 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"leg_alm2map_kernel|leg_map2alm_kernel" -c 2 \
    -o gpurun_out/c4_legendre python tools/profile_run.py --nside 2048 --lmax 4096 > gpurun_out/ncu_leg.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
