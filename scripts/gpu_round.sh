#!/usr/bin/env bash
# One GPU-box pass: GPU tests, smoke, bench, kernel microbench, ncu launch list
# and ncu --set full captures of the top kernels.  Every step is bounded by its
# own timeout and writes into gpurun_out/ so a later failure keeps earlier output.
#   gpurun --timeout 2400 -- bash scripts/gpu_round.sh [steps...]
set -u
mkdir -p gpurun_out
STEPS="${*:-probe tests smoke bench kbench timelines launches ncu}"
log() { echo "== $(date +%T) $*" | tee -a gpurun_out/round.log; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv >> gpurun_out/round.log 2>&1
for s in $STEPS; do
  case $s in
    probe)  log probe;  timeout 300 python scripts/probe_box.py > gpurun_out/probe.log 2>&1; log "probe rc=$?";;
    tests)  log tests;  timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; log "tests rc=$?";;
    smoke)  log smoke;  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; log "smoke rc=$?";;
    bench)  log bench;  timeout 1500 python bench.py --steps 2 --warmup 3 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; log "bench rc=$?";;
    benchfull) log benchfull; timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 --out gpurun_out/bench_full.json > gpurun_out/bench_full.log 2>&1; log "benchfull rc=$?";;
    bench22) log bench22; timeout 2400 python bench.py --config mixtral-8x22b --steps 1 --warmup 3 --warmup-decode 8 --no-cpu-baseline --out gpurun_out/bench22.json > gpurun_out/bench22.log 2>&1; log "bench22 rc=$?";;
    benchref) log benchref; timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1; log "benchref rc=$?";;
    sweep)  log sweep;  timeout 2400 python bench.py --sweep --sweep-decode 8 --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; log "sweep rc=$?";;
    timelines) log timelines
      timeout 300 python scripts/k4v6_timeline.py > gpurun_out/k4v6_timeline.json 2>&1
      timeout 300 python scripts/k3_timeline.py 151 > gpurun_out/k3_timeline.json 2>&1
      timeout 300 python scripts/k4_ce2.py --out gpurun_out/k4_ce2.json > gpurun_out/k4_ce2.log 2>&1
      log "timelines done";;
    benchpa) log benchpa; timeout 1500 python bench.py --policy prefetchall --steps 1 --warmup 3 --decode 32 --warmup-decode 4 --no-cpu-baseline --out gpurun_out/bench_pa.json > gpurun_out/bench_pa.log 2>&1; log "benchpa rc=$?";;
    benchod) log benchod; timeout 1500 python bench.py --policy ondemand --steps 1 --warmup 3 --decode 32 --warmup-decode 4 --no-cpu-baseline --out gpurun_out/bench_od.json > gpurun_out/bench_od.log 2>&1; log "benchod rc=$?";;
    benchor) log benchor; timeout 1500 python bench.py --policy oracle --steps 1 --warmup 3 --decode 32 --warmup-decode 4 --no-cpu-baseline --out gpurun_out/bench_or.json > gpurun_out/bench_or.log 2>&1; log "benchor rc=$?";;
    calib)  log calib;  timeout 900 python scripts/calibrate_cost.py --out gpurun_out/calib.json > gpurun_out/calib.log 2>&1; log "calib rc=$?";;
    kbench) log kbench; timeout 600 python scripts/kbench.py --iters 20 > gpurun_out/kbench.json 2> gpurun_out/kbench.err; log "kbench rc=$?";;
    launches)
      log launches
      DS_LAUNCH_GATE=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
        --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 1 --warmup 1 --decode 4 --warmup-decode 2 --no-cpu-baseline --no-parity --also-22b 0 --calib-requests 1 --calib-decode 4 > gpurun_out/launches.log 2>&1
      log "launches rc=$?"
      python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.md 2>&1;;
    ncuv6)
      log ncuv6
      DS_LAUNCH_GATE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'expert_fused_v6' -s 2 -c 2 \
        -o gpurun_out/k4v6 -f python scripts/kbench.py --only k4 --iters 3 > gpurun_out/ncu_k4v6.log 2>&1
      log "ncu k4v6 rc=$?";;
    ncu)
      log ncu
      DS_LAUNCH_GATE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'expert_fused_v6|staged_gemv|swiglu_gemv|down_gemv' -s 4 -c 4 \
        -o gpurun_out/k4 -f python scripts/kbench.py --only k4 --iters 3 > gpurun_out/ncu_k4.log 2>&1
      log "ncu k4 rc=$?"
      DS_LAUNCH_GATE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'w4_gemm' -s 4 -c 2 \
        -o gpurun_out/k3 -f python scripts/kbench.py --only k3 --iters 3 > gpurun_out/ncu_k3.log 2>&1
      log "ncu k3 rc=$?";;
  esac
done
log done
