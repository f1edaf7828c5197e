# The reference's benchmark suites (micro, miniapp) on the device backend
# through the reference's own API (tests/native/build/device_bench), default
# sizes 2^10..2^24, both precisions, device-resident planes; host planes
# (the reference's DenseVectors staged over PCIe) at a few sizes.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
B=tests/native/build/device_bench
timeout 900 python -m pytest tests/test_adapter.py -q -m gpu > gpurun_out/pytest_adapter.log 2>&1
echo "exit $?" >> gpurun_out/pytest_adapter.log
for s in micro miniapp; do
  for p in f64 f32; do
    timeout 900 $B $s --precision $p --csv gpurun_out/devbench_${s}_${p}.csv > gpurun_out/devbench_${s}_${p}.txt 2>&1
    echo "exit $?" >> gpurun_out/devbench_${s}_${p}.txt
  done
  timeout 900 $B $s --precision f64 --planes host --sizes 1024,65536,1048576,16777216 \
      --csv gpurun_out/devbench_${s}_f64_host.csv > gpurun_out/devbench_${s}_f64_host.txt 2>&1
  echo "exit $?" >> gpurun_out/devbench_${s}_f64_host.txt
done
