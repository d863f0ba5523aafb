#!/bin/bash
# On the GPU box: launch lists (per-kernel device time + DRAM bytes) and one `ncu --set full`
# capture of the top kernel for the bench configurations, summarized on the box by
# tools/ncu_summary.py into gpurun_out/prof/<round>_*.md and ncu_traffic.json (copy to profiles/).
# Every command below first ran without ncu (bench.py exits 0) in the same round.
set -x
mkdir -p gpurun_out/prof
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
R=${ROUND:-r02}
run() {  # cfg, launch-skip, launch-count, full-kernel-regex, full-skip, full-count, traffic class
  cfg=$1
  ncu --metrics $M --clock-control none --csv -s $2 -c $3 --log-file gpurun_out/prof/launches_$cfg.csv \
      python bench.py --config $cfg --no-secondary --steps 1 --warmup 1 > gpurun_out/prof/ncu_$cfg.log 2>&1
  python tools/ncu_summary.py launches gpurun_out/prof/launches_$cfg.csv gpurun_out/prof/${R}_launches_$cfg.md > /dev/null
  ncu --set full --import-source on --clock-control none -k regex:$4 -s $5 -c $6 -o /tmp/full_$cfg \
      python bench.py --config $cfg --no-secondary --steps 1 --warmup 1 > gpurun_out/prof/ncu_full_$cfg.log 2>&1
  python tools/ncu_summary.py full /tmp/full_$cfg.ncu-rep gpurun_out/prof/${R}_ncu_full_$cfg.md > /dev/null
  # traffic per launch from the launch list (every launch of the captured cycles)
  python tools/ncu_summary.py traffic gpurun_out/prof/launches_$cfg.csv gpurun_out/prof/ncu_traffic.json $cfg/$7 $4
  # (the raw report stays on the box: the merged gpurun_out/ is capped at 64 MiB)
  ls -la /tmp/full_$cfg.ncu-rep gpurun_out/prof/launches_$cfg.csv
  gzip -f gpurun_out/prof/launches_$cfg.csv
}
CFGS=${CFGS:-"C2 C3s4 C4"}
for c in $CFGS; do
  case $c in
    C2) run C2 3000 2600 k_arn_step 100 3 arn_step ;;
    C3s4) run C3s4 1200 1200 k_upd 40 2 block_update ;;
    C4) run C4 900 900 k_mgs 30 2 mgs_update ;;
    C5) run C5 1200 1200 k_bupd 40 4 block_update ;;
  esac
done
ls -la gpurun_out/prof
