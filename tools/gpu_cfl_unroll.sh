# The standalone CFL reduction (5R:0W, f64 division/sqrt chains) against
# points per thread (FVB_UNROLL) at several CTA shapes: more independent
# chains per thread against fewer resident warps.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
rm -f gpurun_out/cfl_unroll.jsonl gpurun_out/cfl_unroll_keys.txt
run() {
  key="$1"; shift
  for p in f64 f32; do
    env "$@" timeout 300 python bench.py --config cfl3d --prec $p --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --out gpurun_out/cfl_unroll.jsonl > /dev/null 2>> gpurun_out/cfl_unroll.err
    echo "$key $p" >> gpurun_out/cfl_unroll_keys.txt
  done
}
run default FVB_DUMMY=1
run "128thr minb8 u1" FVB_MODE=2 FVB_THREADS=128 FVB_MINB=8 FVB_UNROLL=1
run "128thr minb4 u2" FVB_MODE=2 FVB_THREADS=128 FVB_MINB=4 FVB_UNROLL=2
run "256thr minb2 u2" FVB_MODE=2 FVB_THREADS=256 FVB_MINB=2 FVB_UNROLL=2
run "256thr minb1 u4" FVB_MODE=2 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=4
run "256thr minb1 u2" FVB_MODE=2 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=2
run "persistent 256 u2" FVB_MODE=1 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=2
run default-again FVB_DUMMY=1
