# The cp.async pipeline CSR form (FVB_CSR_MODE=pipe) against the warp-staged
# default: the CSR parity tests in every mode, then csr_bench.py (7-point
# Laplacian 256^3, L2 flushed between reps) per form and warps per CTA.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k csr > gpurun_out/pytest_csr.log 2>&1
echo "exit $?" >> gpurun_out/pytest_csr.log
rm -f gpurun_out/csr_pipe.jsonl
FVB_CSR_MODE=warp timeout 300 python tools/csr_bench.py --ref-n 0 >> gpurun_out/csr_pipe.jsonl 2>> gpurun_out/csr_pipe.err
for w in 1 2 4; do
  echo "{\"pipe_warps\": $w}" >> gpurun_out/csr_pipe.jsonl
  FVB_CSR_MODE=pipe FVB_CSR_PIPE_WARPS=$w timeout 300 python tools/csr_bench.py --ref-n 0 >> gpurun_out/csr_pipe.jsonl 2>> gpurun_out/csr_pipe.err
done
