#!/bin/bash
# one ncu --set full capture of a kernel (high stall-sampling rate) on a short bench run
# usage: tools/ncu_one.sh TAG KERNEL_REGEX [launch_skip] [count]
TAG=$1; K=$2; SKIP=${3:-60}; CNT=${4:-2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"$K" -s $SKIP -c $CNT \
  -o gpurun_out/one_$TAG python bench.py --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/one_$TAG.log 2>&1; echo "ncu rc=$?"
