set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "stencil" > gpurun_out/pytest_st.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_st.log
timeout 900 python tools/bench_all.py --configs 5 --methods bicgstab,cocr,cors > gpurun_out/bench_st.log 2>&1; echo b=$?
for z in 2 8 16; do CCG_STENCIL_ZC=$z timeout 300 python tools/bench_all.py --configs 5 --methods cocr > gpurun_out/bench_st_zc$z.log 2>&1; done
