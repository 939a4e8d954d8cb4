set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_fused.log
timeout 900 python bench.py --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 --steps 10 --warmup 3 > gpurun_out/bench_fused.log 2>&1
VX_NO_FUSED_SPLAT=1 timeout 900 python bench.py --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 --steps 10 --warmup 3 > gpurun_out/bench_unfused.log 2>&1
for f in fused unfused; do python - $f <<'PY'
import json,sys
l=[x for x in open(f'gpurun_out/bench_{sys.argv[1]}.log') if x.startswith('{')][-1]
d=json.loads(l)
print(sys.argv[1], 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), {k: v for k, v in d['stage_ms'].items()})
PY
done
