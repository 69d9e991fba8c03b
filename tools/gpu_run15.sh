cd $GRAFT_REPO_ROOT
for x in 1 2; do CMG_L1X2=$x timeout 600 python tools/probe_big.py 16384 float32 fast 2>&1 | tail -4 | head -2; done
CMG_L1X2=2 timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or strips" 2>&1 | tail -2
