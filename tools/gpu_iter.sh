# iterate: build, focused GPU tests, panel probe, bench (tail + scans), no CPU legs
set -x
python -m paper_2410_17084_b200.build
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "size_buckets or large_n or config3 or huge or r2 or axis or reference or threshold or stream or sharding or recipe or capacity" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_iter.log
timeout 300 python tools/panel_probe.py --voxels 100000 --reps 3 > gpurun_out/panel_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/panel_probe.log
timeout 600 python bench.py --no-cpu --traj-scans 0 --steps 3 --warmup 3 --scan-reps 10 > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"
