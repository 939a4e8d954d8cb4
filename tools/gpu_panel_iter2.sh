set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q -p no:cacheprovider -k "size_buckets or large_n or config3 or huge or threshold or c05" > gpurun_out/pytest_pi.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pi.log
timeout 300 python tools/panel_probe.py --voxels 100000 --reps 3 > gpurun_out/panel_probe.log 2>&1; cat gpurun_out/panel_probe.log
for C in 1 8; do VX_PANEL_C=$C VX_LIB_PATH=$PWD/build/pt/libvoxgpr.so timeout 300 python tools/panel_phases.py; done
for C in auto 4 8; do if [ $C = auto ]; then unset VX_PANEL_C; else export VX_PANEL_C=$C; fi; timeout 120 python /tmp/cfg3.py > gpurun_out/cfg3_$C.log 2>&1; echo "C=$C"; tail -1 gpurun_out/cfg3_$C.log; done
