#!/bin/bash
# C1 (and C3) call-level A/B of libss variants: tools/sweep.py c1 per variant.
#   gpurun -- 'bash tools/c1ab.sh TAG base,seg512'
TAG=${1:-c1ab}
VARS=${2:-base}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
  for v in ${VARS//,/ }; do
    timeout 600 python tools/sweep.py --configs c1,c3 --variant $v --out /dev/null 2>/dev/null | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/c1ab_$TAG.jsonl
  done
done
echo done
