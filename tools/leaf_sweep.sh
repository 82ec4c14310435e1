cd $GRAFT_REPO_ROOT
for L in 64 96 128 192 256 384; do
  PDG_ND_LEAF=$L timeout 120 python bench.py --steps 10 --warmup 3 --spmv-sizes 256 --spmv-reps 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('A_LEAF', $L, d['value'], d['iterations'][:3], d['phases']['a_solve']['ms_per_step'], d['phases']['flow_solve']['ms_per_step'], d['config']['setup_s'])"
done
for L in 32 64 128 256 512; do
  PDG_ND_FLOW_LEAF=$L timeout 120 python bench.py --steps 10 --warmup 3 --spmv-sizes 256 --spmv-reps 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FLOW_LEAF', $L, d['value'], d['iterations'][:3], d['phases']['a_solve']['ms_per_step'], d['phases']['flow_solve']['ms_per_step'], d['config']['setup_s'])"
done
