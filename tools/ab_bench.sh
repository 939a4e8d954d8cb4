# A/B the library variants under build/<v>/libvoxgpr.so against the in-tree build
# (run on the GPU box from the repo root): tools/ab_bench.sh TAG v1 v2 ...
TAG=$1; shift
python bench.py --no-cpu --traj-scans 0 > gpurun_out/${TAG}_base.log 2>&1
for v in "$@"; do
  VX_LIB_PATH=$PWD/build/$v/libvoxgpr.so python bench.py --no-cpu --traj-scans 0 > gpurun_out/${TAG}_$v.log 2>&1
done
python bench.py --no-cpu --traj-scans 0 > gpurun_out/${TAG}_base2.log 2>&1
