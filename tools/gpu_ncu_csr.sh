# ncu evidence for the CSR accumulation kernel (1 GPU); ncu only after the
# identical plain command exited 0.  Then: python tools/ncu_summary.py r01 csr f64 16777216
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CMD="python tools/csr_bench.py --n 256 --reps 3 --ref-n 0"
$CMD > gpurun_out/ncu_plain_csr.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_csr_f64.csv $CMD > gpurun_out/ncu_launch_csr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:csr_warp -s 1 -c 1 \
    -o gpurun_out/prof_csr_f64 $CMD > gpurun_out/ncu_full_csr.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_csr.log
