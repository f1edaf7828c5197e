cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/hbm_probe tools/hbm_probe.cu && timeout 600 tools/hbm_probe > gpurun_out/hbm_probe.jsonl 2>&1
