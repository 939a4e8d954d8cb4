set -x
python -m paper_2410_17084_b200.build
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_full.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_full.err
