# one GPU round: parity tests, bench (N=1), launch list + ncu captures of the top kernels
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_solve.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for m in split bulk rows; do CCG_GEMV=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$m.log 2>&1; echo bench_$m=$?; tail -1 gpurun_out/bench_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['ah']['achieved'])"; done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
if [ "${NCU:-1}" = 1 ]; then
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_n_split -s 4 -c 1 -o gpurun_out/prof_gemv $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi
