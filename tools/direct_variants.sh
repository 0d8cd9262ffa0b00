#!/bin/bash
# A/B builds of the direct TC kernel's switch (then: python tools/direct_ab.py build/var_s*/libim2win_sm100.so)
set -e
cd "$(dirname "$0")/.."
tools/build_variant.sh s0 -DIM2WIN_DIRECT_SPLIT_BUILD=0 >/dev/null 2>&1 &
tools/build_variant.sh s1 -DIM2WIN_DIRECT_SPLIT_BUILD=1 >/dev/null 2>&1 &
wait
ls build/var_s*/libim2win_sm100.so
