# alm2map host path: median wall over iterations for env-variable variants ("VAR=val,..." tuples)
for v in ${A2M_ENV:-"X=0"}; do
  env $(echo $v | tr , " ") E2E_SKIP_COPY=1 E2E_ITERS=${ITERS:-8} python tools/e2e_probe.py 2>&1 | grep "alm2map wall" | \
    awk '{print $3}' | sort -n | awk -v v="$v" '{a[NR]=$1} END {print v, "median", a[int((NR+1)/2)], "min", a[1], "max", a[NR]}'
done
