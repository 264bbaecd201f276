#!/bin/bash
# One gpurun session: GPU tests, kernel sweep, a bench line, the ncu launch
# list of our kernels, full ncu captures, full-size parity, sharded benches.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG [steps]'
TAG=${1:-r01}
STEPS=${2:-all}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
(nvidia-smi; nproc; lscpu | head -20) > gpurun_out/host_$TAG.txt 2>&1
has() { [[ "$STEPS" == all || ",$STEPS," == *",$1,"* ]]; }
if has test; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
fi
if has kbench; then
  timeout 1200 python tools/kbench.py run --variants ${KB_VARIANTS:-base,mb3,mb5} > gpurun_out/kbench_$TAG.jsonl 2> gpurun_out/kbench_$TAG.err
fi
if has bench; then
  timeout 900 python bench.py --steps 5 --warmup 3 --out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
fi
if has ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quant_kernel|amax_kernel|sums_kernel" -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 3 -c 1 -o gpurun_out/quant_full_$TAG python tools/kbench.py one --variants base --layers 2 --reps 1 --windows=-8:8 > gpurun_out/ncu_full_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 2 -c 1 -o gpurun_out/quant_fused_$TAG python tools/aftrace.py run --variant base --gmode tensor --layers 18 --windows=-8:8 > gpurun_out/ncu_fused_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:amax_kernel -s 3 -c 1 -o gpurun_out/amax_full_$TAG python tools/kbench.py one --variants base --layers 2 --reps 1 --windows=-8:8 > gpurun_out/ncu_amax_$TAG.log 2>&1
  # summarise on the box (each full report with source is ~30 MB; gpurun returns <= 64 MiB)
  for r in quant_full quant_fused amax_full; do
    if [ -f gpurun_out/${r}_$TAG.ncu-rep ]; then
      python tools/ncu_summary.py full gpurun_out/${r}_$TAG.ncu-rep > gpurun_out/${r}_$TAG.md 2>&1
      ncu -i gpurun_out/${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/${r}_$TAG.raw.csv 2>/dev/null
      [ -n "$KEEP_REP" ] && [ "$r" = "$KEEP_REP" ] || rm -f gpurun_out/${r}_$TAG.ncu-rep
    fi
  done
  python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.md 2>&1
fi
if has sweep; then
  timeout 1500 python tools/sweep.py --out gpurun_out/sweep_$TAG.jsonl > gpurun_out/sweep_$TAG.log 2>&1; echo "sweep exit $?" >> gpurun_out/sweep_$TAG.log
fi
if has fullparity; then
  # every block of the BASELINE workloads (and the NEXT rows) against the oracle on the host cores
  timeout 2400 python tools/fullparity.py --configs c2,c4,c3,c5,c5big,c3row,c5fmt --out gpurun_out/fullparity_$TAG.jsonl > gpurun_out/fullparity_$TAG.log 2>&1; echo "fullparity exit $?" >> gpurun_out/fullparity_$TAG.log
fi
if has mrank; then
  # the sharded bench path with 2 ranks sharing the one GPU (gloo carries the amax all-reduce)
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --workload c1_gauss4096 --no-cpu-baseline --dist-backend gloo --out gpurun_out/bench_mrank_$TAG.json > gpurun_out/bench_mrank_$TAG.log 2>&1; echo "mrank exit $?" >> gpurun_out/bench_mrank_$TAG.log
fi
if has nccl1; then
  # the NCCL code path at world size 1 (test-only --force-dist)
  NCCL_DEBUG=WARN timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --steps 3 --warmup 3 --force-dist --no-cpu-baseline --out gpurun_out/bench_nccl1_$TAG.json > gpurun_out/bench_nccl1_$TAG.log 2>&1; echo "nccl1 exit $?" >> gpurun_out/bench_nccl1_$TAG.log
fi
echo done
