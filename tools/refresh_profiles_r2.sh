# Round-2 measurement refresh (GPU box, repo root): bench + reference lines,
# ncu launch list of the config-4 step, ncu --set full of the GPR kernels of
# the config-4 step and of the panel kernel on the tail map.  Summaries are
# written as text; the large .ncu-rep files are removed (gpurun_out <= 64 MiB),
# except the dominant kernel's.
TAG=${1:-r2}
python -m paper_2410_17084_b200.build
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 > gpurun_out/${TAG}_launch_ncu.log 2>&1
python tools/summarize_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gpr_(wdmma|tile)_kernel" -c 7 -o gpurun_out/${TAG}_gpr_full \
    python bench.py --voxels 1000000 --steps 1 --warmup 1 --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 > gpurun_out/${TAG}_full_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_gpr_full.ncu-rep > gpurun_out/${TAG}_ncu_gpr_kernels.txt 2>&1
python tools/ncu_traffic.py gpurun_out/${TAG}_gpr_full.ncu-rep 1000000 > gpurun_out/${TAG}_traffic_main.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gpr_tile_kernel<16" -c 1 -o gpurun_out/${TAG}_dominant \
    python bench.py --voxels 1000000 --steps 1 --warmup 1 --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 > gpurun_out/${TAG}_dom_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_dominant.ncu-rep --page details > gpurun_out/${TAG}_ncu_dominant.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gpr_panel_kernel|k_append|rs_scatter|k_hash_points|gaussians_kernel" -c 8 -o gpurun_out/${TAG}_tail_full \
    python tools/panel_probe.py --voxels 100000 --reps 1 > gpurun_out/${TAG}_tail_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_tail_full.ncu-rep > gpurun_out/${TAG}_ncu_tail_kernels.txt 2>&1
ncu -i gpurun_out/${TAG}_tail_full.ncu-rep --page details -k regex:gpr_panel > gpurun_out/${TAG}_ncu_panel.txt 2>&1
rm -f gpurun_out/${TAG}_gpr_full.ncu-rep gpurun_out/${TAG}_tail_full.ncu-rep
du -sh gpurun_out
echo done
