#!/bin/bash
# Selected parity tests of the in-tree build, then C2 and C5 stream A/B of library builds.
# Usage: AB="libs" AB5="libs" tools/gpu_ab2.sh TAG
TAG=$1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_config_parity.py tests/test_gpu_overlap.py -q -m gpu -x > gpurun_out/pytest_sel_$TAG.log 2>&1; echo "sel rc=$?"; tail -3 gpurun_out/pytest_sel_$TAG.log
timeout 600 bash tools/ab_stream.sh 2 $AB
VM_CONFIG=C5 VM_BLOCKS=400000 VM_RECORDS=40000000 timeout 900 bash tools/ab_stream.sh 2 $AB5
