# One parameterised runner for gpurun calls (run from the repo root on the box):
#   bash tools/gpu.sh tests [pytest args...]     -m gpu tests (default: all)     -> gpurun_out/pytest_gpu.log
#   bash tools/gpu.sh smoke                       __graft_entry__.smoke()         -> gpurun_out/smoke.log
#   bash tools/gpu.sh bench [bench.py args...]    bench.py (N=1)                  -> gpurun_out/bench.log
#   bash tools/gpu.sh ref                         bench.py --impl reference       -> gpurun_out/bench_ref.log
#   bash tools/gpu.sh launches [bench args...]    ncu launch list of bench.py     -> gpurun_out/launches.csv
#   bash tools/gpu.sh ncu <kernel-regex> <count> <python script + args...>
#                                                 ncu --set full capture          -> gpurun_out/prof.ncu-rep
#   bash tools/gpu.sh benchall [args...]          tools/bench_all.py              -> gpurun_out/bench_all.log
#   bash tools/gpu.sh nccl1                       torchrun N=1 bench through NCCL -> gpurun_out/nccl1.log
#   bash tools/gpu.sh round                       tests + smoke + bench + ref + launches
# Several tasks may be chained: bash tools/gpu.sh tests -- bench -- launches
set -u
mkdir -p gpurun_out
run() {
  local task=$1; shift
  case "$task" in
    tests) CCG_PARITY_LOG=gpurun_out/parity.jsonl timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1
           echo "tests rc=$?"; tail -5 gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log ;;
    ref) timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
         tail -1 gpurun_out/bench_ref.log ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
                --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
                > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    ncu) local k=$1 cnt=$2; shift 2
         timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$k" -c "$cnt" -f \
           -o gpurun_out/prof "$@" > gpurun_out/prof.log 2>&1; echo "ncu rc=$?" ;;
    benchall) timeout 2400 python tools/bench_all.py "$@" > gpurun_out/bench_all.log 2>&1; echo "benchall rc=$?" ;;
    nccl1) NCCL_DEBUG=INFO timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
             --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-comm "$@" > gpurun_out/nccl1.log 2>&1
           echo "nccl1 rc=$?"; tail -1 gpurun_out/nccl1.log ;;
    round) run tests; run smoke; run bench; run ref; run launches ;;
    *) echo "unknown task $task"; return 2 ;;
  esac
}
args=("$@")
start=0
for ((i = 0; i <= ${#args[@]}; i++)); do
  if [[ $i -eq ${#args[@]} || "${args[$i]}" == "--" ]]; then
    if (( i > start )); then run "${args[@]:start:i-start}"; fi
    start=$((i + 1))
  fi
done
