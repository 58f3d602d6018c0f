#!/bin/bash
# A/B of the masked pull SpMV at s24 (tools/time_mv.py): row bins (default for
# masked pulls), edge-balanced row tiles, tiles on the degree-ordered layout.
cd "$(dirname "$0")/.."
S=${1:-24}
for d in ${DENSITIES:-0.5}; do
for cfg in "GB_MV_BINS=1" "GB_MV_BINS=0" "GB_MV_BINS=0 GB_MV_ORDERED=1 GB_MV_HOT=0"; do
  echo "== $cfg density $d"
  env $cfg python tools/time_mv.py --scale $S --reps 20 --density $d
done
done
# column stripes (default for structure-only matrices whose vector exceeds 32 MB) vs none
for d in ${DENSITIES:-0.5}; do
for cfg in "GB_MV_STRIPE_BYTES=0" "GB_MV_STRIPE_BYTES=33554432" "GB_MV_STRIPE_BYTES=16777216"; do
  echo "== $cfg density $d"
  env $cfg python tools/time_mv.py --scale $S --reps 20 --density $d
done
done
