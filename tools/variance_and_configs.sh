mkdir -p gpurun_out
for i in 1 2 3 4 5; do timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-all-configs 2>/dev/null | tail -1 > gpurun_out/var_$i.json; done
for w in qwq32b_32k_b4 llama8b_128k_t128 longchat7b_16k; do
  timeout 300 ncu --set full --clock-control none -k regex:prefix_tc -s 3 -c 1 -o gpurun_out/r01e_prefix_$w -f python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-all-configs > /dev/null 2>&1
done
ls gpurun_out | grep -E "var_|r01e_prefix_" 
