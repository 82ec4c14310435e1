# rebuilds the SpMV with different occupancy caps of the prefetch variant and times each
for mb in 3 5 6; do
  touch paper_1801_04984_b200/csrc/spacetime_kp.cu
  make -s -C paper_1801_04984_b200/csrc EXTRA=-DKP_MINB=$mb 2>&1 | tail -2
  echo "== KP_MINB=$mb"
  python bench.py --no-cpu-baseline --config2-n 0 --config4-n 0 --spmv-sizes 256,512,1024 --spmv-reps 50 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/slab',round(d['value'],4),'e2e',round(d['e2e']['value'],4),'spmv phase',d['phases']['spmv']['ms_per_step'], [(s.get('n'),s.get('frac_measured',s.get('frac'))) for s in d['spmv']])
"
done
