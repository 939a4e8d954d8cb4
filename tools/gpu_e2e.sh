set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "engine or capacity or scan_replay or config" > gpurun_out/pytest_e2e.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_e2e.log
timeout 900 python bench.py --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 --steps 10 --warmup 3 > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_e2e.log') if x.startswith('{')][-1]
d=json.loads(l)
print('value', round(d['value']), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'res', round(d['e2e_map_resident']['ms_per_step'],2))
PY
for F in 128 96 64; do VX_PANEL_FROM=$F timeout 900 python bench.py --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 --steps 5 --warmup 3 > gpurun_out/bench_pf$F.log 2>&1; python - $F <<'PY'
import json,sys
l=[x for x in open(f'gpurun_out/bench_pf{sys.argv[1]}.log') if x.startswith('{')][-1]
d=json.loads(l)
print('PANEL_FROM', sys.argv[1], 'ms', round(d['ms_per_step'],2), {k: v for k, v in d['stage_ms'].items() if k in ('gpr_n96','gpr_n128','gpr_n160')})
PY
done
