# e2e (host buffers through the C ABI) of the lighter configs: C2 and the v_mag2 micro-benchmark.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/e2e_more.jsonl
for args in "--config cons2prim1d --prec f64" "--config vmag2 --prec f64" "--config cons2prim1d --prec f32" "--config vmag2 --prec f32"; do
  timeout 600 python bench.py $args --steps 50 --out gpurun_out/e2e_more.jsonl > /dev/null 2>> gpurun_out/e2e_more.err
done
