# map2alm host path: median wall for SHTC_M2A_GROUPS variants (band counts per Legendre launch
# tag; the last tag is split by order chunks), listed space-separated in $M2A_GROUP_LIST
for g in ${M2A_GROUP_LIST:-"1,1,1,1,1,1,1,1"}; do
  SHTC_M2A_GROUPS=$g E2E_SKIP_COPY=1 E2E_ITERS=${ITERS:-8} python tools/e2e_probe.py 2>&1 | grep "map2alm wall" | \
    awk '{print $3}' | sort -n | awk -v v="$g" '{a[NR]=$1} END {print "groups", v, "median", a[int((NR+1)/2)], "min", a[1], "max", a[NR]}'
done
