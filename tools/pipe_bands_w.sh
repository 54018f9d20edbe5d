# host-buffer pair at C4 for "bands|weights" items in $CASES
for c in $CASES; do
  b=${c%%|*}; w=${c#*|}
  for i in 1 2; do
    out=$(SHTC_PIPE_BANDS=$b SHTC_BAND_WEIGHTS=$w E2E_SKIP_COPY=1 python tools/e2e_probe.py 2>&1 | grep "wall")
    echo "$c $(echo "$out" | awk '{print $1, $3}' | tr '\n' ' ')"
  done
done
