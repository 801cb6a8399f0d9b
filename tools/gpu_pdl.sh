set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_pdl.log
for p in 0 1; do CCG_PDL=$p timeout 900 python tools/bench_all.py --configs 2,5,4 --no-dense4 --methods bicgstab,qmr,bicor,cocr,gmres > gpurun_out/bench_pdl$p.log 2>&1; echo b$p=$?; done
for p in 0 1; do CCG_PDL=$p timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_main_pdl$p.log 2>&1; echo m$p=$?; tail -1 gpurun_out/bench_main_pdl$p.log | cut -c1-120; done
