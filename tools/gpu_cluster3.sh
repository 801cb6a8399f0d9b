set -x
mkdir -p gpurun_out
for cs in 2 4 8 16; do CCG_CLUSTER_SIZE=$cs timeout 300 python tools/bench_all.py --configs 1 --methods bicgstab,cgne > gpurun_out/b1_cs$cs.log 2>&1; echo cs$cs; cut -c1-170 gpurun_out/b1_cs$cs.log; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cluster_solve -c 1 -o gpurun_out/prof_cluster python tools/bench_all.py --configs 1 --reps 1 --methods bicgstab > gpurun_out/ncu_cl.log 2>&1; echo ncu=$?
