# Legendre timing of the shipped library and of tuning variants (paper_1106_0159_b200/_build/var_<name>,
# built with build.build_variant) listed in $VARS
python tools/variant_bench.py 2>&1 | tail -1
for v in ${VARS:-smem shfl_m3 shfl_m4}; do SHTC_VARIANT_LIB=paper_1106_0159_b200/_build/var_$v/libshtc.so timeout 300 python tools/variant_bench.py 2>&1 | tail -1; done
