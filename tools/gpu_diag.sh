set -x
VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so timeout 120 python tools/diag_bench.py
for C in 1 2; do VX_PANEL_C=$C timeout 300 python tools/panel_probe.py --voxels 100000 --reps 2; done
timeout 900 python bench.py --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 --steps 20 --warmup 5 > gpurun_out/bench_e2e20.log 2>&1
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_e2e20.log') if x.startswith('{')][-1]
d=json.loads(l)
print('value', round(d['value']), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'res', round(d['e2e_map_resident']['ms_per_step'],2), d['clocks'])
PY
