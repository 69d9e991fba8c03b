cd $GRAFT_REPO_ROOT
timeout 600 python tools/probe_big.py 16384 float32 fast
CMG_FUSED=0 timeout 600 python tools/probe_big.py 16384 float32 fast
timeout 600 python tools/probe_big.py 8192 float64 exact
timeout 600 python tools/probe_big.py 8192 float64 fast
