VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so timeout 120 python tools/diag_bench.py
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "size_buckets or large_n or config3" 2>&1 | tail -2
timeout 300 python tools/panel_probe.py --voxels 100000 --reps 2
timeout 120 python /tmp/cfg3.py | tail -2
