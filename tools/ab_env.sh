#!/bin/bash
# A/B of environment settings on one library build: the stream device period
# (tools/stream_probe.py), settings alternating.  Usage: tools/ab_env.sh rounds "ENV=.." "ENV=.." ...
R=$1; shift
for r in $(seq $R); do
  for E in "$@"; do
    echo -n "[$E] "; env $E python tools/stream_probe.py 2>/dev/null | grep "Engine.fuse_frame"
  done
done
