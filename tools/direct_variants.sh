#!/bin/bash
# A/B builds of the direct TC kernel's switches: tools/direct_variants.sh  (then run tools/direct_ab.py on the box)
set -e
cd "$(dirname "$0")/.."
tools/build_variant.sh d00 -DIM2WIN_DIRECT_PAD_PITCH=0 -DIM2WIN_DIRECT_SPLIT_BUILD=0 >/dev/null 2>&1 &
tools/build_variant.sh d01 -DIM2WIN_DIRECT_PAD_PITCH=0 -DIM2WIN_DIRECT_SPLIT_BUILD=1 >/dev/null 2>&1 &
wait
tools/build_variant.sh d10 -DIM2WIN_DIRECT_PAD_PITCH=1 -DIM2WIN_DIRECT_SPLIT_BUILD=0 >/dev/null 2>&1 &
tools/build_variant.sh d11 -DIM2WIN_DIRECT_PAD_PITCH=1 -DIM2WIN_DIRECT_SPLIT_BUILD=1 >/dev/null 2>&1 &
wait
ls build/var_d*/libim2win_sm100.so
