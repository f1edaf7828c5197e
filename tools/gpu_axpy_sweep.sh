# C1 (axpy-sin, N=1e6, latency-bound) launch-shape sweep, f64 and f32.
# Usage (under gpurun): bash tools/gpu_axpy_sweep.sh [warm|cold]
#   warm: K steps back to back in one CUDA graph (--l2-warm; the round-1 sweep)
#   cold: the bench default, L2 flushed between individually timed steps
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
L2=--l2-warm; STEPS=2000
if [ "${1:-warm}" = cold ]; then L2=; STEPS=300; fi
rm -f gpurun_out/axpy_sweep.jsonl gpurun_out/axpy_sweep_keys.txt
for cfg in "0 0 0 0" "2 256 2 0" "2 256 2 2" "2 256 2 1" "2 128 2 0" "2 128 2 2" "2 256 1 0" "2 512 1 0" "2 256 1 1" "2 128 1 0"; do
  set -- $cfg
  for p in f64 f32; do
    if [ "$1" = 0 ]; then
      timeout 300 python bench.py --config axpy --prec $p --steps $STEPS --warmup 20 $L2 --no-e2e --no-cpu-baseline --out gpurun_out/axpy_sweep.jsonl > /dev/null 2>> gpurun_out/axpy_sweep.err
    else
      FVB_MODE=$1 FVB_THREADS=$2 FVB_MINB=$3 FVB_VEC=$4 timeout 300 python bench.py --config axpy --prec $p --steps $STEPS --warmup 20 $L2 --no-e2e --no-cpu-baseline --out gpurun_out/axpy_sweep.jsonl > /dev/null 2>> gpurun_out/axpy_sweep.err
    fi
    echo "mode=$1 threads=$2 minb=$3 vec=$4 $p" >> gpurun_out/axpy_sweep_keys.txt
  done
done
