# ncu evidence for the headline kernel (1 GPU).  Each ncu command runs only
# after the identical plain command exited 0 in this call.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CFG="${1:-flux3d}"; PREC="${2:-f64}"; N="${3:-20000000}"
CMD="python bench.py --config $CFG --prec $PREC --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --n $N"
$CMD > gpurun_out/ncu_plain_${CFG}_${PREC}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${CFG}_${PREC}.csv $CMD > gpurun_out/ncu_launch_${CFG}_${PREC}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pointwise_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${CFG}_${PREC} $CMD > gpurun_out/ncu_full_${CFG}_${PREC}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_${CFG}_${PREC}.log
