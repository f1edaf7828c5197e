# C1 cold (bench default) against groups per thread (FVB_UNROLL) and CTA shape.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/c1_unroll.jsonl gpurun_out/c1_unroll_keys.txt
for cfg in "0 0 0 0" "2 256 2 2" "2 256 1 2" "2 256 1 4" "2 128 1 2" "2 256 1 1"; do
  set -- $cfg
  for p in f64 f32; do
    if [ "$1" = 0 ]; then
      timeout 300 python bench.py --config axpy --prec $p --steps 300 --no-cpu-baseline --out gpurun_out/c1_unroll.jsonl > /dev/null 2>> gpurun_out/c1_unroll.err
    else
      FVB_MODE=$1 FVB_THREADS=$2 FVB_MINB=$3 FVB_UNROLL=$4 timeout 300 python bench.py --config axpy --prec $p --steps 300 --no-cpu-baseline --out gpurun_out/c1_unroll.jsonl > /dev/null 2>> gpurun_out/c1_unroll.err
    fi
    echo "mode=$1 threads=$2 minb=$3 unroll=$4 $p" >> gpurun_out/c1_unroll_keys.txt
  done
done
