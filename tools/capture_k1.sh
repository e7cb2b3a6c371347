#!/bin/bash
# The profiling recipe of the headline kernel, run on the GPU box (gpurun -- 'bash tools/capture_k1.sh r02'):
#   1. bench.py without a profiler (the numbers that count), 2. the ncu launch list of the same command,
#   3. one `ncu --set full` capture of K1, 4. summaries + profiles/roofline.json (stamped with the source hash).
# Everything lands in gpurun_out/; copy what is to be judged into profiles/.
set -u
tag=${1:-rXX}
out=gpurun_out
mkdir -p $out
cmd="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 1"
$cmd > $out/bench_${tag}_plain.json 2> $out/bench_${tag}_plain.err || { echo "bench failed"; tail -5 $out/bench_${tag}_plain.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_${tag}_k1.csv $cmd > $out/ncu_list_${tag}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 3 -c 1 -f -o $out/prof_${tag}_k1 $cmd > $out/ncu_full_${tag}.log 2>&1
python tools/ncu_summary.py $out/prof_${tag}_k1.ncu-rep --title "K1 ($tag): $cmd" --roofline $out/roofline_${tag}.json > $out/ncu_${tag}_k1.txt
echo "captured: $out/bench_${tag}_plain.json $out/launches_${tag}_k1.csv $out/ncu_${tag}_k1.txt $out/roofline_${tag}.json"
