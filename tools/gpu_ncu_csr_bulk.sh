cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export FVB_CSR_MODE=bulk
CMD="python tools/csr_bench.py --n 256 --reps 3 --ref-n 0"
$CMD > gpurun_out/ncu_plain_csrbulk.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_bulk -s 1 -c 1 \
    -o gpurun_out/prof_csr_bulk $CMD > gpurun_out/ncu_full_csrbulk.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_csrbulk.log
