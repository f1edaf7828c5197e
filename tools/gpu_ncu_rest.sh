cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_ncu.sh vmag2 f64 50000000
bash tools/gpu_ncu.sh vmag2 f32 50000000
bash tools/gpu_ncu.sh cons2prim1d f32 50000000
