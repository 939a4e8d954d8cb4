# large-n panel kernel: correctness + timing (run on the GPU box from the repo root)
set -x
python -m paper_2410_17084_b200.build
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "size_buckets or large_n or config3 or huge" > gpurun_out/pytest_large.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_large.log
for C in auto 1 2; do
  if [ "$C" = auto ]; then unset VX_PANEL_C; else export VX_PANEL_C=$C; fi
  timeout 600 python bench.py --no-cpu --traj-scans 0 --steps 3 --warmup 3 --scan-reps 10 > gpurun_out/large_$C.log 2>&1; echo "bench $C rc=$?"
done
unset VX_PANEL_C
VX_OLD_BIG=1 timeout 600 python bench.py --no-cpu --traj-scans 0 --steps 3 --warmup 3 --scan-reps 10 > gpurun_out/large_old.log 2>&1; echo "bench old rc=$?"
