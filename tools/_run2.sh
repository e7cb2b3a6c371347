python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "refined_tier" 2>&1 | tail -3
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/k1_sweep.py run 2>&1 | tail -2
P='import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        r=json.loads(l); print(r["name"], r["mode"], "ms", round(r["ms"],4), "ids", r["ids"], "stats", r["stats_collected"], "ok", r["oracle_counts_equal"], r["oracle_pairs_equal"])'
for sub in 0 1 2; do
  echo "tier_sub=$sub"; GJ_DEBUG_PLAN=1 GJ_TIER_SUB=$sub GJ_HIST_REP=0 GJ_NODE_PAL_MAX_MB=0 python tools/bench_configs.py 4 --scale 0.04 --dir16-level 17 2>gpurun_out/plan_$sub.log | python -c "$P"; grep "32-bit tier" gpurun_out/plan_$sub.log | head -1
done
echo auto; GJ_DEBUG_PLAN=1 GJ_HIST_REP=0 GJ_NODE_PAL_MAX_MB=0 python tools/bench_configs.py 4 --scale 0.04 --dir16-level 17 2>gpurun_out/plan_auto.log | python -c "$P"; grep "32-bit tier" gpurun_out/plan_auto.log | head -1
echo cfg2-auto; GJ_DEBUG_PLAN=1 python tools/bench_configs.py 2 --no-stats 2>gpurun_out/plan_c2.log | python -c "$P"; grep "32-bit tier" gpurun_out/plan_c2.log | head -1
echo cfg3-auto; GJ_DEBUG_PLAN=1 python tools/bench_configs.py 3 --no-stats 2>gpurun_out/plan_c3.log | python -c "$P"; grep "32-bit tier" gpurun_out/plan_c3.log | head -1
