#!/bin/bash
# pipelined host-path timelines at C4: comma tuples "a2m_mode,band_group,bands,m2a_mode" in $VARIANTS
for v in ${VARIANTS:-2,1,8,2}; do
  IFS=, read -r am bg nb mm <<< "$v"
  echo "== a2m-mode $am band-group $bg bands $nb m2a-mode $mm"
  SHTC_PIPE_MODE=$am SHTC_M2A_BAND_GROUP=$bg SHTC_PIPE_BANDS=$nb SHTC_M2A_MODE=$mm SHTC_PIPE_TRACE=1 \
    python tools/e2e_probe.py 2>&1 | grep -v "^dev\|^h2d\|^d2h\|^both" | tail -4
done
