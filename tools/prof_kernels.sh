set -e
KERNELS=("$@")
python bench.py --steps 1 --warmup 1 --no-cpu --traj-scans 0 > gpurun_out/p_plain.log 2>&1
for k in "${KERNELS[@]}"; do
  tag=$(echo "$k" | tr -cd 'a-z0-9_')
  ncu --set full --kernel-name-base demangled --import-source on --clock-control none -k "regex:$k" -c 1 -o gpurun_out/p_$tag \
     python bench.py --steps 1 --warmup 1 --no-cpu --traj-scans 0 > gpurun_out/p_$tag.log 2>&1 || true
done
