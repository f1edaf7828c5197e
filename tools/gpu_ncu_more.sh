cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_ncu.sh flux3d f32 20000000
bash tools/gpu_ncu.sh jacobian3d f32 10000000
bash tools/gpu_ncu.sh axpy f64 1000000
