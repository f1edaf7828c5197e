cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/c1.jsonl
for p in f64 f32; do
timeout 300 python bench.py --config axpy --prec $p --steps 200 --warmup 5 --no-cpu-baseline --out gpurun_out/c1.jsonl > /dev/null 2>> gpurun_out/c1.err
timeout 300 python bench.py --config axpy --prec $p --steps 1000 --warmup 5 --l2-warm --no-cpu-baseline --out gpurun_out/c1.jsonl > /dev/null 2>> gpurun_out/c1.err
done
