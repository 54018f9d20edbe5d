# A/B of the ring-stage times: shipped library vs $VARS variants, interleaved, 3 rounds
for i in 1 2 3; do
  echo "== default"; python tools/profile_run.py --nside 2048 --lmax 4096 --iters 3 2>&1 | tail -2 | grep -o "^[a-z2]* {'legendre_ms': [0-9.]*, 'fft_ms': [0-9.]*"
  for v in $VARS; do echo "== $v"; SHTC_VARIANT_LIB=paper_1106_0159_b200/_build/var_$v/libshtc.so python tools/profile_run.py --nside 2048 --lmax 4096 --iters 3 2>&1 | tail -2 | grep -o "^[a-z2]* {'legendre_ms': [0-9.]*, 'fft_ms': [0-9.]*"; done
done
