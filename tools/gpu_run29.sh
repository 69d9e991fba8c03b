cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_variants.py -m gpu -q 2>&1 | grep -E "passed|failed|mismatch" | head -20
