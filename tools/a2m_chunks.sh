# alm2map from pinned memory at C4 for a_lm chunk counts in $CHUNKS and head-band counts in $HEADS
for c in ${CHUNKS:-4}; do for h in ${HEADS:-2}; do
  for i in 1 2 3; do
    out=$(SHTC_A2M_CHUNKS=$c SHTC_A2M_HEAD=$h E2E_SKIP_COPY=1 python tools/e2e_probe.py 2>&1 | grep "alm2map wall")
    echo "chunks $c head $h $(echo "$out" | awk '{print $3}' | tr '\n' ' ')"
  done
done; done
