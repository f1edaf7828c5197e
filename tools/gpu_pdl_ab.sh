# A/B of programmatic dependent launch (FVB_PDL=0 vs the default) on one box:
# C1 as an L2-warm CUDA graph of 1000 steps and cold, the adapter's captured
# time step at n = 1024, and the default flux bench line.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/pdl_ab.jsonl
for pdl in 0 1; do
  for p in f64 f32; do
    FVB_PDL=$pdl timeout 300 python bench.py --config axpy --prec $p --steps 1000 --l2-warm --no-cpu-baseline --out gpurun_out/pdl_ab.jsonl > /dev/null 2>> gpurun_out/pdl_ab.err
    echo "{\"pdl\": $pdl, \"what\": \"axpy warm $p\"}" >> gpurun_out/pdl_ab.jsonl
  done
  FVB_PDL=$pdl timeout 300 python bench.py --config axpy --prec f64 --steps 300 --no-cpu-baseline --out gpurun_out/pdl_ab.jsonl > /dev/null 2>> gpurun_out/pdl_ab.err
  echo "{\"pdl\": $pdl, \"what\": \"axpy cold f64\"}" >> gpurun_out/pdl_ab.jsonl
  FVB_PDL=$pdl timeout 300 python bench.py --steps 100 --no-e2e --no-cpu-baseline --out gpurun_out/pdl_ab.jsonl > /dev/null 2>> gpurun_out/pdl_ab.err
  echo "{\"pdl\": $pdl, \"what\": \"flux default\"}" >> gpurun_out/pdl_ab.jsonl
  FVB_PDL=$pdl tests/native/build/device_acceptance overhead | sed "s/^{/{\"pdl\": $pdl, /" >> gpurun_out/pdl_ab.jsonl
done
