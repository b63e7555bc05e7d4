#!/bin/bash
# run-to-run determinism stress of the persistent attention kernels (all head dims, odd / even tile counts,
# every forward variant)
for shp in "1 1024 1 64" "1 256 4 64" "2 640 2 128" "4 2048 8 128" "2 1920 3 112" "3 1152 5 96"; do
  for v in 2 3 4; do
    LYNX_ATTN_FWD_TILES=$v timeout 300 python tools/attn_race.py 200 $shp 2>&1 | tail -1 | sed "s/^/fwd$v $shp: /"
  done
done
