#!/bin/bash
# One parametrised GPU-box runner (replaces the round-1 one-off gpu_run*.sh).
# Companions: ab.sh / e2e_ab.sh (single-GPU library-variant A/B), mgpu_ab.sh
# (multi-GPU A/B, any bench args e.g. --placement 0/1/2), sweep.sh /
# sweep_ab.sh (BASELINE config 5), shim_timing.sh, nvlink_probe.sh.
#   scripts/gpu.sh <task> [args]    run under gpurun, writes to gpurun_out/
# tasks:
#   tests            pytest -m gpu (one GPU), then smoke()
#   bench [args]     bench.py (N=1) + the reference arm, JSON to gpurun_out/bench_*.json
#   mgpu N [args]    bench.py under torchrun on N GPUs
#   mtests N         the multi-GPU pytest cases on N GPUs
#   ncu REGEX [args] ncu --set full of the first 3 launches matching REGEX in bench.py [args]
#   launches [args]  ncu launch list (gpu__time_duration.sum) of bench.py [args]
#   sanitize TOOL CMD...  compute-sanitizer --tool TOOL on one command
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
task=$1; shift
case "$task" in
  tests)
    timeout 1500 python -m pytest tests -m gpu -x -q -rs "$@" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
    tail -3 gpurun_out/gpu_tests.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
    tail -2 gpurun_out/smoke.log ;;
  bench)
    nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
    timeout 900 python bench.py "$@" > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err; echo "bench rc=$?"
    timeout 900 python bench.py --impl reference "$@" > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
    echo "ref rc=$?"; tail -c 600 gpurun_out/bench_g1.err ;;
  mgpu)
    n=$1; shift
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus "$n" "$@" > gpurun_out/bench_g$n.json 2> gpurun_out/bench_g$n.err
    echo "mgpu rc=$?"; tail -c 600 gpurun_out/bench_g$n.err ;;
  mtests)
    n=$1; shift
    timeout 1500 python -m pytest tests/test_multi_gpu.py -m gpu -x -q -s "$@" > gpurun_out/mgpu_tests_g$n.log 2>&1
    echo "mtests rc=$?"; tail -5 gpurun_out/mgpu_tests_g$n.log ;;
  ncu)
    re=$1; shift
    timeout 600 python bench.py "$@" > gpurun_out/ncu_plain.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$re" -s 2 -c 1 \
      -o gpurun_out/prof_$(echo "$re" | tr -c 'a-zA-Z0-9_' _) -f python bench.py "$@" > gpurun_out/ncu.log 2>&1
    echo "ncu rc=$?"; tail -5 gpurun_out/ncu.log ;;
  launches)
    timeout 600 python bench.py "$@" > gpurun_out/launches_plain.log 2>&1 && \
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py "$@" > gpurun_out/launches_ncu.log 2>&1
    echo "launches rc=$?" ;;
  sanitize)
    tool=$1; shift
    timeout 1500 compute-sanitizer --tool "$tool" --error-exitcode 9 "$@" > gpurun_out/sanitize_$tool.log 2>&1
    echo "sanitize $tool rc=$?"; tail -5 gpurun_out/sanitize_$tool.log ;;
  *) echo "unknown task $task"; exit 2 ;;
esac
