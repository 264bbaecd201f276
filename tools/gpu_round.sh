#!/bin/bash
# One gpurun session: GPU tests, a bench line, the ncu launch list and one
# full ncu capture of the quantize kernel.  Usage (from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1; nproc >> gpurun_out/nvsmi_$TAG.txt; lscpu | head -20 >> gpurun_out/nvsmi_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 20 -c 1 -o gpurun_out/quant_full_$TAG python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amax_kernel -s 20 -c 1 -o gpurun_out/amax_full_$TAG python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_amax_$TAG.log 2>&1
echo done
