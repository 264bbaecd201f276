mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 3 -c 1 -o gpurun_out/quant_r0_k python tools/kbench.py one --variants base --layers 2 --reps 1 --windows=0:0 > gpurun_out/ncu_r0_k.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_kernel -s 3 -c 1 -o gpurun_out/quant_r8_k python tools/kbench.py one --variants base --layers 2 --reps 1 --windows=-8:8 > gpurun_out/ncu_r8_k.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --out gpurun_out/bench_k.json > gpurun_out/bench_k.log 2>&1
