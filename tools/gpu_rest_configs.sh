# The remaining entry points of SURVEY §8a (prim->cons, primitive flux, EOS,
# standalone CFL) on one GPU: one bench line each (with e2e and the
# reference beside it), then the ncu launch list + one --set full capture per
# f64 kernel (tools/gpu_ncu.sh; summarise with tools/ncu_summary.py).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
OUT=gpurun_out/rest_configs.jsonl
rm -f $OUT
for c in prim2cons3d flux_prim3d eos cfl3d; do
  for p in f64 f32; do
    timeout 600 python bench.py --config $c --prec $p --steps 100 --out $OUT > /dev/null 2>> gpurun_out/rest_configs.err
  done
done
if [ "$1" = ncu ]; then
  for c in prim2cons3d flux_prim3d eos cfl3d; do bash tools/gpu_ncu.sh $c f64 20000000; done
fi
if [ "$1" = ncu ]; then
  # summarise on the box (the full captures are too large to bring back)
  python tools/ncu_summary.py r01 prim2cons3d f64 20000000 flux_prim3d f64 20000000 \
      eos f64 20000000 cfl3d f64 20000000 > gpurun_out/ncu_summary_rest.log 2>&1
  mkdir -p gpurun_out/profiles_rest
  cp profiles/r01_prim2cons3d_f64.json profiles/r01_flux_prim3d_f64.json profiles/r01_eos_f64.json \
     profiles/r01_cfl3d_f64.json profiles/traffic.json gpurun_out/profiles_rest/ 2>> gpurun_out/ncu_summary_rest.log
  rm -f gpurun_out/prof_*.ncu-rep
fi
