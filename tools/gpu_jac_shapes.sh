# Launch shapes of the 3-D Jacobian + CFL kernel (75 outputs; the default,
# 32-byte accesses and one 256-thread CTA per SM, runs at 248 registers):
# narrower accesses and more resident CTAs.  Keys in jac_shapes_keys.txt.
# FVB_VEC counts elements per access: f64 4 = 32 B (default), 2 = 16 B,
# 1 = 8 B; f32 8 = 32 B, 4 = 16 B.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
rm -f gpurun_out/jac_shapes.jsonl gpurun_out/jac_shapes_keys.txt
run() {
  key="$1"; p="$2"; shift 2
  env "$@" timeout 300 python bench.py --config jacobian3d --prec $p --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --out gpurun_out/jac_shapes.jsonl > /dev/null 2>> gpurun_out/jac_shapes.err
  echo "$key $p" >> gpurun_out/jac_shapes_keys.txt
}
for p in f64 f32; do
  if [ $p = f64 ]; then H=2; else H=4; fi
  run default $p FVB_DUMMY=1
  run "16B minb2" $p FVB_MODE=2 FVB_THREADS=256 FVB_UNROLL=1 FVB_MINB=2 FVB_VEC=$H
  run "16B minb4" $p FVB_MODE=2 FVB_THREADS=256 FVB_UNROLL=1 FVB_MINB=4 FVB_VEC=$H
  run "16B 128thr minb2" $p FVB_MODE=2 FVB_THREADS=128 FVB_UNROLL=1 FVB_MINB=2 FVB_VEC=$H
  run "32B 128thr minb2" $p FVB_MODE=2 FVB_THREADS=128 FVB_UNROLL=1 FVB_MINB=2
  run "32B 128thr minb4" $p FVB_MODE=2 FVB_THREADS=128 FVB_UNROLL=1 FVB_MINB=4
  run "32B persistent" $p FVB_MODE=1 FVB_THREADS=256 FVB_UNROLL=1 FVB_MINB=1
  run default-again $p FVB_DUMMY=1
done
run "8B minb2" f64 FVB_MODE=2 FVB_THREADS=256 FVB_UNROLL=1 FVB_MINB=2 FVB_VEC=1
