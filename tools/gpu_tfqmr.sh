set -x
mkdir -p gpurun_out
timeout 900 python tools/bench_all.py --configs 1,2,3,5,4 --no-dense4 --methods tfqmr > gpurun_out/bench_tfqmr.log 2>&1; echo b=$?; cut -c1-220 gpurun_out/bench_tfqmr.log
