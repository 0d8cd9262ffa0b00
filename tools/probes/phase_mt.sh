for mt in 1 2 4; do echo "MT=$mt"; IM2WIN_PHASE_MT=$mt timeout 120 python tools/tc_kernels.py conv4 128 2>&1 | tail -2 | cut -c1-60; done
