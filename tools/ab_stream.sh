#!/bin/bash
# A/B of library builds on one box: the back-to-back stream device period
# (tools/stream_probe.py's Engine.fuse_frame leg), builds alternating.
# Usage: tools/ab_stream.sh rounds libA.so libB.so [libC.so ...]
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    echo -n "$(basename $L): "; VOXMESH_B200_LIB=$L python tools/stream_probe.py 2>/dev/null | grep "Engine.fuse_frame"
  done
done
