set -x
python -m paper_2410_17084_b200.build
timeout 300 python tools/debug_stream.py > gpurun_out/debug_stream.log 2>&1; echo "dbg rc=$?"
cat gpurun_out/debug_stream.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_all.log
