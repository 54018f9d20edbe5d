# host-buffer transforms at C4 for band-weight lists in $WEIGHTS (space separated; "-" = default):
# one line per run with the alm2map and map2alm wall-clock ms
for w in ${WEIGHTS:--}; do
  for i in 1 2 3; do
    if [ "$w" = "-" ]; then out=$(E2E_SKIP_COPY=1 python tools/e2e_probe.py 2>&1 | grep wall);
    else out=$(SHTC_BAND_WEIGHTS=$w E2E_SKIP_COPY=1 python tools/e2e_probe.py 2>&1 | grep wall); fi
    echo "$w $(echo "$out" | awk '{print $1, $3}' | tr '\n' ' ')"
  done
done
