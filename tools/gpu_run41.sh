cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -n 3
python tools/time_big.py 16384 float32 fast 1 '[{}, {"CMG_DBG": "65536"}, {"CMG_L1X2": "1"}, {"CMG_L1X2": "1", "CMG_DBG": "65536"}, {"CMG_L1X2": "7"}]'
python tools/time_big.py 512 float32 fast 64 '[{}, {"CMG_DBG": "65536"}]'
