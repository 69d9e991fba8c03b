cd $GRAFT_REPO_ROOT
export CMG_FUSED=0
for d in 0 8 1 2 4 3 7; do CMG_DBG=$d timeout 120 python tools/time_levels.py exact; done
CMG_DBG=0 timeout 120 python tools/time_levels.py fast
CMG_DBG=8 timeout 120 python tools/time_levels.py fast
