cd $GRAFT_REPO_ROOT
export CMG_FUSE_MASK=1
timeout 900 python -m pytest tests -m gpu -q -x -k "energy or small or c3 or batch" 2>&1 | tail -1
for nb in 148 296 592 1184; do CMG_ENERGY_CTAS=$nb timeout 300 python tools/stamps_report.py fast float32 | grep -E "per cycle|energy"; done
