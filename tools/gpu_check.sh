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
  for cfg in "256 1 1" "256 2 1" "128 1 1" "128 4 1" "128 1 2" "256 1 2" "512 1 1" "256 2 2"; do
    set -- $cfg
    FVB_THREADS=$1 FVB_MINB=$2 FVB_UNROLL=$3 timeout 300 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline --out gpurun_out/sweep.jsonl > /dev/null 2>> gpurun_out/sweep.err
    echo "threads=$1 minb=$2 unroll=$3" >> gpurun_out/sweep_keys.txt
  done
fi
