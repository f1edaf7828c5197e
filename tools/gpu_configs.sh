# Every BASELINE config on one GPU (+ the paper's v_mag2 micro-benchmark),
# optionally with the HBM mix probe.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
OUT=gpurun_out/configs.jsonl
rm -f $OUT
if [ "$1" = probe ]; then
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/hbm_probe tools/hbm_probe.cu && tools/hbm_probe > gpurun_out/hbm_probe.jsonl 2>&1
fi
for args in "--config flux3d --prec f64" "--config flux3d --prec f32" "--config cons2prim1d --prec f64" "--config cons2prim1d --prec f32" \
            "--config jacobian3d --prec f64 --no-e2e" "--config jacobian3d --prec f32 --no-e2e" \
            "--config axpy --prec f64 --steps 300" "--config axpy --prec f64 --steps 1000 --l2-warm" "--config vmag2 --prec f64" "--config vmag2 --prec f32"; do
  timeout 600 python bench.py $args --out $OUT > /dev/null 2>> gpurun_out/configs.err
done
