cd $GRAFT_REPO_ROOT
for t in 2 3; do echo "f32 tma=$t"; CMG_TMA=$t timeout 300 python -m pytest tests -m gpu -q -x -k "c3_f32in" 2>&1 | tail -1; done
for t in 2 3; do echo "f64 tma=$t"; CMG_TMA=$t timeout 300 python -m pytest tests -m gpu -q -x -k "c3_f64" 2>&1 | tail -1; done
