# Round-end measurement refresh (run on the GPU box from the repo root):
#   bench line, reference-arm line, ncu launch list, ncu --set full of the GPR kernels.
set -e
TAG=${1:-r1}
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu --traj-scans 0 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --traj-scans 0 > gpurun_out/${TAG}_launch_ncu.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gpr_(wdmma|tile|big)_kernel" -c 7 -o gpurun_out/${TAG}_gpr_full \
    python bench.py --steps 1 --warmup 1 --no-cpu --traj-scans 0 > gpurun_out/${TAG}_full_ncu.log 2>&1
