# Round-2 final measurement refresh (GPU box, repo root): bench + reference
# lines, ncu launch list of the config-4 step, ncu --set full summaries of the
# GPR kernels, the dominant kernel (details page), the n<=16 warp kernel, the
# hash-stage kernels and the panel kernel on the tail map.  Large .ncu-rep
# files are removed (gpurun_out <= 64 MiB).
TAG=${1:-r2}
set -x
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0 > gpurun_out/${TAG}_launch_ncu.log 2>&1
python tools/summarize_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1
B="python bench.py --voxels 1000000 --steps 1 --warmup 1 --no-cpu --traj-scans 0 --scan-reps 0 --tail-voxels 0"
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gpr_(wdmma|tile)_kernel" -c 7 -o gpurun_out/${TAG}_gpr_full $B > gpurun_out/${TAG}_full_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_gpr_full.ncu-rep > gpurun_out/${TAG}_ncu_gpr_kernels.txt 2>&1
python tools/ncu_traffic.py gpurun_out/${TAG}_gpr_full.ncu-rep 1000000 > gpurun_out/${TAG}_traffic_main.json 2>&1
ncu -i gpurun_out/${TAG}_gpr_full.ncu-rep --page details -k "regex:tile_kernel<.int.16," > gpurun_out/${TAG}_ncu_dominant.txt 2>&1
ncu -i gpurun_out/${TAG}_gpr_full.ncu-rep --page details -k "regex:wdmma_kernel<.int.16>" > gpurun_out/${TAG}_ncu_wdmma16.txt 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:k_hash_points|k_place|k_point_rank|k_seg_append|k_first_flags|k_rank_slots|gaussians_kernel|k_pca_prepass" -c 8 \
    -o gpurun_out/${TAG}_hbm $B > gpurun_out/${TAG}_hbm_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_hbm.ncu-rep > gpurun_out/${TAG}_ncu_hbm_stages.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:gpr_panel_kernel" -c 1 -o gpurun_out/${TAG}_panel \
    python tools/panel_probe.py --voxels 100000 --reps 1 > gpurun_out/${TAG}_panel_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_panel.ncu-rep > gpurun_out/${TAG}_ncu_panel_summary.txt 2>&1
ncu -i gpurun_out/${TAG}_panel.ncu-rep --page details > gpurun_out/${TAG}_ncu_panel.txt 2>&1
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
echo done
