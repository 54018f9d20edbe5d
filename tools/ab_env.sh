# A/B of the C4 device-resident stage times for environment settings in $ENVS ("-" = none), 3 rounds
for i in 1 2 3; do
  for e in ${ENVS:--}; do
    if [ "$e" = "-" ]; then out=$(python tools/profile_run.py --nside 2048 --lmax 4096 --iters 3 2>&1 | tail -2);
    else out=$(env $e python tools/profile_run.py --nside 2048 --lmax 4096 --iters 3 2>&1 | tail -2); fi
    echo "$e $(echo "$out" | grep -o "'legendre_ms': [0-9.]*, 'fft_ms': [0-9.]*" | tr '\n' ' ')"
  done
done
