python tools/dbg/k9_flaky.py c4 0 25 2000 2>&1 | tail -1 | cut -c1-140
POLY_L2_KEEP_MB=0,32 python tools/dbg/k9_flaky.py c4 0 25 2000 2>&1 | tail -1 | cut -c1-140
POLY_L2_KEEP_MB=32,32 python tools/dbg/k9_flaky.py c4 0 25 1000 2>&1 | tail -1 | cut -c1-140
