cd $GRAFT_REPO_ROOT
export CMG_FUSE_MASK=1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/stamps_report.py exact float64
timeout 300 python tools/stamps_report.py fast float32
