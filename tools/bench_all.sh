mkdir -p gpurun_out
for w in c1_gauss4096 c3_act_student_t c4_llama70b_kv c5_gauss_1gib; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --e2e-steps 1 --out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1
  echo "$w exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']
print('  value %.0f GB/s  step %.3f ms  frac %.3f  exec %s  e2e %s  cpu %s  launches %d' % (d['value'], d['ms_per_step'], r['frac'], r.get('executed_frac'), d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'), d['gpu_launches']))" 2>&1 | tail -1
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -c 600 gpurun_out/bench_ref.log
