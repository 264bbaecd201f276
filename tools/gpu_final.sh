#!/bin/bash
# Round-end evidence on one B200 (TAG names the files):
#   the bench line, the ncu launch list of the bench command, ncu --set full
#   captures of the bench's top kernel (a mid-chain trailing-amax launch) and of the
#   plain search kernel (device amax) with DRAM traffic, the configs sweep
#   (+ oracle samples) and its counting run, sanitizers.
#   gpurun --timeout 5400 -- 'bash tools/gpu_final.sh r02 [steps]'
TAG=${1:-r02}
STEPS=${2:-all}
mkdir -p gpurun_out
has() { [[ "$STEPS" == all || ",$STEPS," == *",$1,"* ]]; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
(nvidia-smi; nproc; lscpu | head -20) > gpurun_out/host_$TAG.txt 2>&1
if has bench; then
  timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1
fi
if has ncu; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quant_kernel|amax_kernel|sums_kernel|rowscale_kernel|dequant" -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.md 2>&1
  # a mid-chain launch of the bench's trailing-amax chain: quant launch 4 of 8
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 4 -c 1 \
    -o gpurun_out/quant_fused_$TAG python tools/chainprof.py --chain-only > gpurun_out/ncu_fused_$TAG.log 2>&1
  # DRAM bytes of every launch of the chain -> profiles/quant_traffic.json "trail" (bench.py's traffic field)
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:quant_kernel --csv --log-file gpurun_out/chain_traffic_$TAG.csv python tools/chainprof.py --chain-only > gpurun_out/chain_traffic_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 1 -c 1 \
    -o gpurun_out/quant_plain_$TAG python tools/qone.py --workload c2_qwen3_8b_weights --tensors 28 --window=-8:8 --reps 2 > gpurun_out/ncu_plain_$TAG.log 2>&1
  for r in quant_fused quant_plain; do
    if [ -f gpurun_out/${r}_$TAG.ncu-rep ]; then
      python tools/ncu_summary.py full gpurun_out/${r}_$TAG.ncu-rep > gpurun_out/${r}_$TAG.md 2>&1
      python tools/ncu_summary.py hot gpurun_out/${r}_$TAG.ncu-rep >> gpurun_out/${r}_$TAG.md 2>&1
      ncu -i gpurun_out/${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/${r}_$TAG.raw.csv 2>/dev/null
      ncu -i gpurun_out/${r}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_$TAG.sass.csv 2>/dev/null
      rm -f gpurun_out/${r}_$TAG.ncu-rep
    fi
  done
fi
if has sweep; then
  timeout 2400 python tools/sweep.py --out gpurun_out/sweep_$TAG.jsonl > gpurun_out/sweep_$TAG.log 2>&1; echo "sweep exit $?" >> gpurun_out/sweep_$TAG.log
  python tools/kbench.py build --variants count > /dev/null 2>&1
  timeout 1500 python tools/sweep.py --configs c1,c2,c3,c4,c5 --c5-gib 1 --variant count --out gpurun_out/sweep_count_$TAG.jsonl > gpurun_out/sweep_count_$TAG.log 2>&1
fi
if has test; then
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
fi
if has sanitize; then
  bash tools/sanitize.sh > gpurun_out/sanitize_$TAG.log 2>&1
fi
echo done
