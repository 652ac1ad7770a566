#!/bin/bash
# Round measurement bundle (run under gpurun; writes gpurun_out/<tag>_*):
#   full bench line (all configs, cpu_baseline), clocks during it, the ncu launch list of a short
#   bench run, and one `ncu --set full` capture each of the prefix and tree/merge kernels.
# usage: tools/profile_round.sh TAG
cd "$(dirname "$0")/.."
T=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap \
    --format=csv -lms 200 > $O/${T}_clocks.csv &
SMI=$!
python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
kill $SMI
cat $O/${T}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-configs > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefix_tc -s 3 -c 1 -o $O/${T}_prefix -f \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-configs > $O/${T}_ncu_prefix.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tree_merge -s 3 -c 1 -o $O/${T}_treemerge -f \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-configs > $O/${T}_ncu_tm.log 2>&1
tail -3 $O/${T}_ncu_prefix.log
ls -la $O | grep $T
