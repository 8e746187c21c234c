python tools/dbg/k9_flaky.py c4 0 25 3000 2>&1 | tail -1 | cut -c1-160
POLY_L2_KEEP_MB=0,32 python tools/dbg/k9_flaky.py c4 0 25 1000 2>&1 | tail -1 | cut -c1-160
python tools/dbg/k9_flaky.py c2s 0 25 1500 2>&1 | tail -1 | cut -c1-160
python tools/dbg/k9_flaky.py c3s 0 25 1500 2>&1 | tail -1 | cut -c1-160
python tools/dbg/k9_flaky.py c2 0 25 500 2>&1 | tail -1 | cut -c1-160
POLY_K1_KEEP_MB=0 python tools/dbg/k9_flaky.py c2 0 25 500 2>&1 | tail -1 | cut -c1-160
python tools/dbg/k9_flaky.py c3 0 10 300 2>&1 | tail -1 | cut -c1-160
