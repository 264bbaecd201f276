#!/bin/bash
# ncu --set full captures with the per-CUDA-source-line and per-SASS-line
# pages exported as CSV (instruction attribution), summarised on the box.
#   gpurun -- 'bash tools/gpu_src.sh TAG "c5_gauss_1gib:0:0 c5_gauss_1gib:-8:8" [variant]'
TAG=${1:-src}
CASES=${2:-"c5_gauss_1gib:0:0"}
VAR=${3:-base}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
[ "$VAR" != base ] && python tools/kbench.py build --variants $VAR >> gpurun_out/build_$TAG.log 2>&1
for c in $CASES; do
  IFS=: read -r wl lo hi <<< "$c"
  name=${wl}_${lo}_${hi}_$TAG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quant_kernel|quant_narrow" -s 1 -c 1 \
    -o gpurun_out/$name python tools/qone.py --workload $wl --window=$lo:$hi --reps 2 --variant $VAR > gpurun_out/$name.log 2>&1
  if [ -f gpurun_out/$name.ncu-rep ]; then
    python tools/ncu_summary.py full gpurun_out/$name.ncu-rep > gpurun_out/$name.md 2>&1
    python tools/ncu_summary.py hot gpurun_out/$name.ncu-rep >> gpurun_out/$name.md 2>&1
    ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source cuda > gpurun_out/$name.cuda.csv 2>&1
    ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>&1
    rm -f gpurun_out/$name.ncu-rep
  fi
done
echo done
