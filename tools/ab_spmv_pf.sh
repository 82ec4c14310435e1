# A/B of the SpMV variants: header prefetch (PDG_SPMV_PF), QK-last block order (PDG_SPMV_QLAST), PK blocks first (PDG_SPMV_PKFIRST)
for v in "0 0 0" "1 1 0" "1 1 1" "1 1 0" "1 1 1"; do
  set -- $v
  echo "== PDG_SPMV_PF=$1 PDG_SPMV_QLAST=$2 PDG_SPMV_PKFIRST=$3"
  PDG_SPMV_PF=$1 PDG_SPMV_QLAST=$2 PDG_SPMV_PKFIRST=$3 python bench.py --no-cpu-baseline --config2-n 0 --config4-n 0 --spmv-sizes ${SIZES:-256,512,1024} --spmv-reps 50 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/slab',round(d['value'],4),'e2e',round(d['e2e']['value'],4),'spmv phase',d['phases']['spmv']['ms_per_step'], [(s.get('n'),s.get('frac_measured',s.get('frac'))) for s in d['spmv']])
"
done
