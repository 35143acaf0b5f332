timeout 900 python -m pytest tests/test_solver_gpu.py tests/test_baselines_gpu.py tests/test_distributed_gpu.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --skip-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['time_to_converge'])
for c,v in d.get('configs',{}).items(): print(c, v['sweep_ms'], {a:(v[a]['seconds'],v[a]['iterations'],v[a]['t_eig']) for a in ('hoscf','ihoscf') if a in v})"
timeout 600 python tools/solve_probe.py C2 C5 --alg hoscf,ihoscf --reps 2 2>&1 | grep rep1
