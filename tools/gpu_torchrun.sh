# The torchrun launch path of bench.py at N=1 (the driver's N>1 command
# shape): NCCL init, barriers, max-over-ranks, the CFL allreduce.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517"
$TR bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/tr_flux.json 2> gpurun_out/tr_flux.err; echo "exit $?" >> gpurun_out/tr_flux.err
$TR bench.py --gpus 1 --steps 10 --warmup 3 --config jacobian3d --no-e2e > gpurun_out/tr_jac.json 2> gpurun_out/tr_jac.err; echo "exit $?" >> gpurun_out/tr_jac.err
$TR bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/tr_ref.json 2> gpurun_out/tr_ref.err; echo "exit $?" >> gpurun_out/tr_ref.err
