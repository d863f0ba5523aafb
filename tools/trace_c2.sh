#!/bin/bash
# raw per-phase trace lines of the block-iteration kernel (C2), plus the phase table
cd "$GRAFT_REPO_ROOT" || exit 1
o=gpurun_out/trace_c2; mkdir -p $o
for r in 1 2; do echo "$(python tools/time_c2.py 5 2>&1 | tail -1)"; done > $o/time.log 2>&1
SKC_TRACE_ORTH=1 python tools/time_c2.py 1 2> $o/trace.err > /dev/null
python tools/phase_breakdown.py $o/trace.err > $o/phases.md 2>&1
grep "^\[step k=5\]" $o/trace.err | head -40 | tail -6 > $o/raw.txt; grep "^\[step k=9\]" $o/trace.err | head -40 | tail -3 >> $o/raw.txt
grep "^\[skew" $o/trace.err | head -300 | tail -9 >> $o/raw.txt
rm -f $o/trace.err
cat $o/time.log $o/raw.txt; head -24 $o/phases.md
