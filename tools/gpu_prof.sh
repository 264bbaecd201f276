#!/bin/bash
# ncu --set full captures (with source-level stall attribution) of the search
# kernel on chosen workloads / windows, summarised on the box.
#   gpurun -- 'bash tools/gpu_prof.sh TAG "c3_act_student_t:0:0 c5_gauss_8gib:-1:1 ..." [fused]'
TAG=${1:-prof}
CASES=${2:-"c3_act_student_t:0:0"}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
for c in $CASES; do
  IFS=: read -r wl lo hi <<< "$c"
  name=${wl}_${lo}_${hi}_$TAG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 1 -c 1 \
    -o gpurun_out/$name python tools/qone.py --workload $wl --window=$lo:$hi --reps 2 > gpurun_out/$name.log 2>&1
  if [ -f gpurun_out/$name.ncu-rep ]; then
    python tools/ncu_summary.py full gpurun_out/$name.ncu-rep > gpurun_out/$name.md 2>&1
    python tools/ncu_summary.py hot gpurun_out/$name.ncu-rep >> gpurun_out/$name.md 2>&1
    rm -f gpurun_out/$name.ncu-rep
  fi
done
if [ -n "$3" ]; then
  name=c2_fused_r8_$TAG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 2 -c 1 \
    -o gpurun_out/$name python tools/aftrace.py run --variant base --gmode tensor --layers 18 --windows=-8:8 > gpurun_out/$name.log 2>&1
  if [ -f gpurun_out/$name.ncu-rep ]; then
    python tools/ncu_summary.py full gpurun_out/$name.ncu-rep > gpurun_out/$name.md 2>&1
    python tools/ncu_summary.py hot gpurun_out/$name.ncu-rep >> gpurun_out/$name.md 2>&1
    rm -f gpurun_out/$name.ncu-rep
  fi
fi
# timings of the same cases without the profiler
for c in $CASES; do
  IFS=: read -r wl lo hi <<< "$c"
  timeout 300 python tools/qone.py --workload $wl --window=$lo:$hi --reps 5 >> gpurun_out/qone_$TAG.jsonl 2>>gpurun_out/qone_$TAG.err
done
echo done
