# The ncu launch list of the default bench command (1 GPU), after the same
# command exited 0 without ncu in this call.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/launchlist_plain.json 2> gpurun_out/launchlist_plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench_default.csv $CMD > gpurun_out/launchlist_ncu.log 2>&1
echo "exit $?" >> gpurun_out/launchlist_ncu.log
