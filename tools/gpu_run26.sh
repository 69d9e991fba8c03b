cd $GRAFT_REPO_ROOT
export CMG_FUSE_MASK=1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
CMG_FUSED_FINALIZE=0 timeout 300 python tools/stamps_report.py fast float32 | grep -E "per cycle|energy|finalize|cond"
for nb in 148 512 1184 2368; do CMG_ENERGY_CTAS=$nb timeout 300 python tools/stamps_report.py fast float32 | grep -E "energy"; done
