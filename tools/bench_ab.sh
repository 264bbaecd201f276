#!/bin/bash
# Bench-level A/B: the current libss.so against libss_prev.so, alternating,
# each `bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline`.
#   gpurun -- 'bash tools/bench_ab.sh TAG [rounds]'
TAG=${1:-bab}
R=${2:-3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2605_12464_b200/libss.so /tmp/libss_cur.so
for i in $(seq $R); do
  for v in cur prev; do
    if [ $v = cur ]; then cp /tmp/libss_cur.so paper_2605_12464_b200/libss.so; else cp paper_2605_12464_b200/libss_prev.so paper_2605_12464_b200/libss.so; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'v': '$v', 'value': d['value'], 'ms': d['ms_per_step']}))" >> gpurun_out/bench_ab_$TAG.jsonl
  done
done
cp /tmp/libss_cur.so paper_2605_12464_b200/libss.so
echo done
