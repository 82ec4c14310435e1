#!/bin/bash
# k_nd_stream unit-count sweep at config 2 (32^3): PDG_ND_STREAM_UNITS = minimum units per level
for u in 0 1500 3000 6000 12000; do
  echo "== PDG_ND_STREAM_UNITS=$u"
  PDG_ND_STREAM_UNITS=$u timeout 600 python tools/config2_probe.py 32 3 2>&1 | tail -2
done
