# C4 end to end (fvb_jacobian_host, pinned, N = 2.5e7 f64) against the host
# side's thread counts and where the 18 duplicate entries travel
# (host copies vs PCIe).  Keys in gpurun_out/e2e_jac_keys.txt.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
rm -f gpurun_out/e2e_jac.jsonl gpurun_out/e2e_jac_keys.txt
run() {
  key="$1"; shift
  env "$@" timeout 600 python bench.py --config jacobian3d --prec f64 --steps 5 --warmup 3 --e2e-steps 5 \
      --e2e-points 25000000 --no-cpu-baseline --out gpurun_out/e2e_jac.jsonl > /dev/null 2>> gpurun_out/e2e_jac.err
  echo "$key" >> gpurun_out/e2e_jac_keys.txt
}
run default FVB_DUMMY=1
run "fill 4" FVB_FILL_THREADS=4
run "fill 12" FVB_FILL_THREADS=12
run "fill 16" FVB_FILL_THREADS=16
run "pool 7" FVB_POOL_THREADS=7
run "pool 7 fill 8" FVB_POOL_THREADS=7 FVB_FILL_THREADS=8
run "dups on link" FVB_DUPS_ON_LINK=1
run "dups on link fill 12" FVB_DUPS_ON_LINK=1 FVB_FILL_THREADS=12
run default-again FVB_DUMMY=1
