set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 3 -c 1 -f -o gpurun_out/prof_r01_k1_final2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01_k1_final2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_ncu_list.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 | cut -c1-200
