timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_config_parity.py tests/test_gpu_overlap.py -q -m gpu -x > gpurun_out/pytest_sel_$1.log 2>&1; echo "sel rc=$?"; tail -3 gpurun_out/pytest_sel_$1.log
timeout 600 bash tools/ab_stream.sh 3 $AB
