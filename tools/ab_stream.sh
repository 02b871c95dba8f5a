#!/bin/bash
# A/B of two library builds on one box: the back-to-back stream device period
# (tools/stream_probe.py's Engine.fuse_frame leg), alternating A and B.
# Usage: tools/ab_stream.sh libA.so libB.so [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for L in $A $B; do
    echo -n "$(basename $L): "; VOXMESH_B200_LIB=$L python tools/stream_probe.py 2>/dev/null | grep "Engine.fuse_frame"
  done
done
