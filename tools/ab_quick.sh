# Quick A/B of library variants on the config-4 step (GPU box, repo root):
#   tools/ab_quick.sh TAG v1 v2 ...   (build/<v>/libvoxgpr.so; "tree" = in-tree build)
TAG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = tree ]; then unset VX_LIB_PATH; else export VX_LIB_PATH=$PWD/build/$v/libvoxgpr.so; fi
  timeout 600 python bench.py --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 --steps 5 --warmup 3 > gpurun_out/${TAG}_${v}_$rep.log 2>&1
  python - "$v" gpurun_out/${TAG}_${v}_$rep.log <<'PY'
import json, sys
ls = [l for l in open(sys.argv[2]) if l.startswith("{")]
if not ls:
    print(sys.argv[1], "FAILED"); sys.exit()
d = json.loads(ls[-1])
print(f"{sys.argv[1]:10s} {d['ms_per_step']:7.2f} ms", {k: round(v, 2) for k, v in d["stage_ms"].items() if v})
PY
done
done
unset VX_LIB_PATH
