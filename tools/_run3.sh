python tools/fullsize.py 4 --scale 0.04 --points 100000000 --variants --save-index /tmp/gj_full4_test.gjx --check 1000000 --host-points 0 2>&1 | grep -v "^{" | tail -20
python tools/fullsize.py 4 --scale 1.0 --variants --save-index /tmp/gj_full4.gjx --check 0 --host-points 0 --out gpurun_out/full4_variants.json > gpurun_out/full4_variants.log 2>&1
grep "fullsize\]\|\[gj\] K1 32" gpurun_out/full4_variants.log | tail -30
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_read.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --kernel-name regex:join_kernel -c 3 --csv --log-file gpurun_out/full4_ncu.csv python tools/fullsize.py 4 --scale 1.0 --load-index /tmp/gj_full4.gjx --reps 1 --check 0 --host-points 0 > gpurun_out/full4_ncu.log 2>&1
tail -3 gpurun_out/full4_ncu.log | cut -c1-300
rm -f /tmp/gj_full4.gjx /tmp/gj_full4_test.gjx
