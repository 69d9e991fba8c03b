cd $GRAFT_REPO_ROOT
CMG_FUSE_MASK=1 timeout 300 python tools/stamps_report.py exact float64
CMG_FUSE_MASK=1 timeout 300 python tools/stamps_report.py fast float32
CMG_FUSE_MASK=7 timeout 300 python tools/stamps_report.py fast float32
