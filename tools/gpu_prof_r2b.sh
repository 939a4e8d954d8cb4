# Profiling pass (session 2 of round 2): tile-kernel phase cycles (diagnostics
# build) and source-level ncu of the n<=16 warp kernel and the n<=128 tile kernel.
set -x
VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so timeout 300 python tools/phase_timing.py > gpurun_out/phase_timing.log 2>&1; echo "phase rc=$?"
cat gpurun_out/phase_timing.log
for K in "gpr_wdmma_kernel<16>" "gpr_tile_kernel<16"; do
  tag=$(echo "$K" | tr -cd 'a-z0-9')
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$K" -c 1 -o gpurun_out/src_$tag \
    python bench.py --voxels 1000000 --steps 1 --warmup 1 --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 > gpurun_out/src_$tag.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i gpurun_out/src_$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$tag.csv 2>/dev/null
  ncu -i gpurun_out/src_$tag.ncu-rep --page details > gpurun_out/src_${tag}_details.txt 2>&1
  python tools/ncu_lines.py gpurun_out/src_$tag.csv 60 > gpurun_out/src_${tag}_lines.txt 2>&1
  gzip -f gpurun_out/src_$tag.csv
  rm -f gpurun_out/src_$tag.ncu-rep
done
du -sh gpurun_out
