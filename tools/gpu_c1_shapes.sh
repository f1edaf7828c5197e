# C1 (axpy-sin, N=1e6) cold-step launch shapes against wave quantisation:
# the default one-shot grid is 977 CTAs over 148 SMs x 4 resident (1.65
# waves); persistent grid-stride grids of one wave, and 128-thread tiles with
# more resident CTAs.  L2 flushed between individually timed steps (bench
# default).  Keys in gpurun_out/c1_shapes_keys.txt, lines in c1_shapes.jsonl.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
rm -f gpurun_out/c1_shapes.jsonl gpurun_out/c1_shapes_keys.txt
run() {  # key, env...
  key="$1"; shift
  for p in f64 f32; do
    env "$@" timeout 300 python bench.py --config axpy --prec $p --steps 300 --warmup 20 --no-e2e --no-cpu-baseline --out gpurun_out/c1_shapes.jsonl > /dev/null 2>> gpurun_out/c1_shapes.err
    echo "$key $p" >> gpurun_out/c1_shapes_keys.txt
  done
}
run default FVB_DUMMY=1
run "persistent 256x1 occ" FVB_MODE=1 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=1
run "persistent 256x1 cap3" FVB_MODE=1 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=1 FVB_CTAS=3
run "persistent 256x1 cap2" FVB_MODE=1 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=1 FVB_CTAS=2
run "persistent 256x2 occ" FVB_MODE=1 FVB_THREADS=256 FVB_MINB=1 FVB_UNROLL=2
run "tiles 128x1 minb4" FVB_MODE=2 FVB_THREADS=128 FVB_MINB=4 FVB_UNROLL=1
run "tiles 128x1 minb8" FVB_MODE=2 FVB_THREADS=128 FVB_MINB=8 FVB_UNROLL=1
run "tiles 128x2 minb4" FVB_MODE=2 FVB_THREADS=128 FVB_MINB=4 FVB_UNROLL=2
run "tiles 256x1 minb4" FVB_MODE=2 FVB_THREADS=256 FVB_MINB=4 FVB_UNROLL=1
run "tiles 256x2 minb2" FVB_MODE=2 FVB_THREADS=256 FVB_MINB=2 FVB_UNROLL=2
