#!/bin/bash
# Round-end evidence for one build (run under gpurun): bench lines of every workload, the reference arm, the ncu launch
# list and one --set full capture per kernel.  usage: tools/final_measure.sh <tag>
R=${1:-r2}
O=gpurun_out
python bench.py --steps 10 --warmup 3 > $O/${R}_bench_c3.json 2> $O/${R}_bench_c3.err
python bench.py --impl reference --steps 1 --warmup 0 > $O/${R}_bench_c3_reference.json 2> $O/${R}_bench_c3_reference.err
python bench.py --workload c1 --steps 20 --warmup 3 --no-cpu > $O/${R}_bench_c1.json 2>/dev/null
python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c2.json 2>/dev/null
python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c4.json 2>/dev/null
python bench.py --workload c3q --steps 10 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c5_10k.json 2>/dev/null
python bench.py --workload c3q --scale 3 --steps 10 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c5_29k.json 2>/dev/null
python bench.py --workload c5 --scale 2 --steps 5 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c5_117k.json 2>/dev/null
python bench.py --workload c5 --scale 4 --steps 5 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c5_233k.json 2>/dev/null
python bench.py --workload c5 --scale 17 --steps 3 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c5_1m.json 2>/dev/null
python bench.py --workload c5 --scale 34 --steps 3 --warmup 3 --no-cpu --no-latency > $O/${R}_bench_c5_2m.json 2>/dev/null
bash tools/capture_all.sh $R
for f in $O/${R}_bench_*.json; do echo "$f: $(head -c 300 $f)"; done
