# host-buffer pair at C4 for pipeline band counts in $BANDS (3 runs each, warm-up run dropped)
for b in ${BANDS:-8}; do
  for i in 1 2; do
    out=$(SHTC_PIPE_BANDS=$b E2E_SKIP_COPY=1 python tools/e2e_probe.py 2>&1 | grep "wall")
    echo "bands $b $(echo "$out" | awk '{print $1, $3}' | tr '\n' ' ')"
  done
done
