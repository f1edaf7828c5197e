cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_ncu.sh flux3d f64 20000000
bash tools/gpu_ncu.sh jacobian3d f64 10000000
bash tools/gpu_ncu.sh cons2prim1d f64 50000000
