# Launch shapes of the standalone CFL reduction (5R:0W, f64 and f32).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
rm -f gpurun_out/cfl_sweep.jsonl gpurun_out/cfl_sweep_keys.txt
for cfg in "0 0 0 0" "2 256 4 0" "2 128 2 0" "2 128 4 0" "2 128 8 0" "2 128 1 0"; do
  set -- $cfg
  for p in f64 f32; do
    if [ "$1" = 0 ]; then
      timeout 300 python bench.py --config cfl3d --prec $p --steps 100 --no-cpu-baseline --out gpurun_out/cfl_sweep.jsonl > /dev/null 2>> gpurun_out/cfl_sweep.err
    else
      FVB_MODE=$1 FVB_THREADS=$2 FVB_MINB=$3 FVB_VEC=$4 timeout 300 python bench.py --config cfl3d --prec $p --steps 100 --no-cpu-baseline --out gpurun_out/cfl_sweep.jsonl > /dev/null 2>> gpurun_out/cfl_sweep.err
    fi
    echo "mode=$1 threads=$2 minb=$3 vec=$4 $p" >> gpurun_out/cfl_sweep_keys.txt
  done
done
