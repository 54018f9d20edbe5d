# map2alm host-path variants: "mode,chunks" tuples in $M2A_VARIANTS
for v in ${M2A_VARIANTS:-0,8 2,8}; do IFS=, read -r m c <<< "$v"
 echo "mode $m chunks $c"; SHTC_M2A_CHUNKS=$c SHTC_M2A_MODE=$m SHTC_PIPE_TRACE=1 E2E_SKIP_COPY=1 E2E_ITERS=3 python tools/e2e_probe.py 2>&1 | grep "pipe map2alm\|map2alm wall" | tail -2
done
