#!/bin/bash
# A/B on the box: tools/time_c2.py under each value of one environment switch
#   VAR=SKC_ORTH_PFL2 VALS="0 1 2" bash tools/ab_env.sh
cd "$GRAFT_REPO_ROOT" || exit 1
o=gpurun_out/ab_env; mkdir -p $o
for r in 1 2; do
  for v in $VALS; do echo "$VAR=$v: $(env $VAR=$v python tools/time_c2.py 5 2>&1 | tail -1)"; done
done > $o/$VAR.log 2>&1
cat $o/$VAR.log
