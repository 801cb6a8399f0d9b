set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_next.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "pbicgstab or next3 or sharded_cfg1 or replicated_cfg1" > gpurun_out/pytest_pb.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_pb.log
timeout 900 python tools/bench_all.py --configs 1,2,3,5,4 --no-dense4 --methods pbicgstab,bicgstab > gpurun_out/bench_pb.log 2>&1; echo b=$?
