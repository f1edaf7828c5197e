# GPU-box check: parity tests, one bench line, a launch-tuning sweep.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tests|bench|sweep|all]
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
what="${1:-all}"
(nvidia-smi; nproc; free -g; lscpu | head -20) > gpurun_out/box.txt 2>&1
if [ "$what" = tests ] || [ "$what" = all ]; then
  timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if [ "$what" = bench ] || [ "$what" = all ]; then
  timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
  timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
if [ "$what" = sweep ] || [ "$what" = all ]; then
  rm -f gpurun_out/sweep.jsonl gpurun_out/sweep_keys.txt
  for cfg in "2 256 1 0" "2 256 2 0" "2 256 4 0" "2 128 1 0" "2 128 2 0" "2 512 1 0" "2 256 2 2" "2 256 4 2" "1 256 1 0" "1 256 2 0"; do
    set -- $cfg
    for c in "flux3d --prec f64" "flux3d --prec f32" "jacobian3d --prec f64"; do
      FVB_MODE=$1 FVB_THREADS=$2 FVB_UNROLL=$3 FVB_VEC=$4 timeout 300 python bench.py --config $c --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --out gpurun_out/sweep.jsonl > /dev/null 2>> gpurun_out/sweep.err
      echo "mode=$1 threads=$2 unroll=$3 vec=$4 $c" >> gpurun_out/sweep_keys.txt
    done
  done
fi
