set -x
python -m paper_2410_17084_b200.build
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q -p no:cacheprovider -k "size_buckets or large_n or config3 or huge or r2 or axis or reference or threshold or stream" > gpurun_out/pytest_r2.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2.log
timeout 300 python tools/panel_probe.py --voxels 100000 --reps 3 > gpurun_out/panel_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/panel_probe.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gpr_panel_kernel -s 1 -c 1 -o gpurun_out/panel_full python tools/panel_probe.py --voxels 100000 --reps 2 > gpurun_out/ncu_panel.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_panel.log
