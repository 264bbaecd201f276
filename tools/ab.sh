#!/bin/bash
# A/B of libss builds on the box: kbench (C2 subset, device amax) and qone
# (C5 1 GiB) per variant, alternating, then the GPU tests and one bench line
# of the current build.
#   gpurun -- 'bash tools/ab.sh TAG "old,base" [tests]'
TAG=${1:-ab}
VARS=${2:-old,base}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
for rep in 1 2; do
  for v in ${VARS//,/ }; do
    timeout 600 python tools/kbench.py one --variants $v --layers 4 --reps 10 --windows=0:0,-1:1,-2:2,-2:6,-8:8 >> gpurun_out/kbench_$TAG.jsonl 2>> gpurun_out/kbench_$TAG.err
    for wl in c5_gauss_1gib c1_gauss4096; do
      for w in 0:0 -1:1 -2:2 -8:8; do
        timeout 300 python tools/qone.py --workload $wl --window=$w --reps 20 --variant $v 2>>gpurun_out/qone_$TAG.err | sort -t: -k5 | python -c "import sys,json; L=[json.loads(l) for l in sys.stdin]; L.sort(key=lambda d: d['ms']); print(json.dumps(L[len(L)//2]))" | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/qone_$TAG.jsonl
      done
    done
  done
done
if [ -n "$3" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
  timeout 900 python bench.py --steps 5 --warmup 3 --out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
fi
echo done
