python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/ozaki_check.py 2>&1 | tail -8
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['value'], d['result_check'], {k:(v['ms_per_launch'],v['launches']) for k,v in d['stages'].items() if 'ozaki' in k or k in ('recon_residual','slice_svd','gram_syrk')})"
python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4', d['value'])"
