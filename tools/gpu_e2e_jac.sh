# e2e (host buffers through fvb_jacobian_host) of C4 on a bounded 2.5e7-point slice.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/e2e_jac.jsonl
for p in f64 f32; do
  timeout 900 python bench.py --config jacobian3d --prec $p --steps 20 --e2e-points 25000000 --out gpurun_out/e2e_jac.jsonl > /dev/null 2>> gpurun_out/e2e_jac.err
done
