# CSR forms on one B200: the CSR parity/bounds tests, then each form through
# tools/csr_bench.py (7-point Laplacian, 256^3).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "csr" > gpurun_out/pytest_csr.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_csr.log
rm -f gpurun_out/csr_modes.jsonl
for m in row warp; do
  FVB_CSR_MODE=$m timeout 300 python tools/csr_bench.py --n 256 --reps 20 --ref-n 0 >> gpurun_out/csr_modes.jsonl 2>> gpurun_out/csr_modes.err
done
for u in 2 4; do
  FVB_CSR_MODE=warp FVB_CSR_UNROLL=$u timeout 300 python tools/csr_bench.py --n 256 --reps 20 --ref-n 0 | sed "s/\"kernel\": \"csr_warp/\"kernel\": \"csr_warp_unroll$u/" >> gpurun_out/csr_modes.jsonl 2>> gpurun_out/csr_modes.err
done
