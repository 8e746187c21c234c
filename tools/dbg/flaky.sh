R=${1:-80}
python tools/dbg/k9_flaky.py c4 0 25 $R 2>&1 | tail -1
python tools/dbg/k9_flaky.py c4 4 25 $R 2>&1 | tail -1      # no PDL
python tools/dbg/k9_flaky.py c4 2 25 $R 2>&1 | tail -1      # no graph
POLY_NO_EPI=1 python tools/dbg/k9_flaky.py c4 0 25 $R 2>&1 | tail -1
POLY_L2_KEEP_MB=0,0 python tools/dbg/k9_flaky.py c4 0 25 $R 2>&1 | tail -1
POLY_NO_TILED=1 python tools/dbg/k9_flaky.py c4 0 25 $R 2>&1 | tail -1
python tools/dbg/k9_flaky.py c4 0 25 $R 2>&1 | tail -1
