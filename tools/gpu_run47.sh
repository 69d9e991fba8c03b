cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -n 3
python tools/time_big.py 16384 float32 fast 1 '[{}, {"CMG_ROWPAIR": "3"}, {"CMG_ROWPAIR": "3", "CMG_RP_PIPE": "1"}, {"CMG_ROWPAIR": "3", "CMG_RP_PIPE": "1", "CMG_TS3": "16"}]'
python tools/time_big.py 512 float32 fast 64 '[{}, {"CMG_ROWPAIR": "3", "CMG_RP_PIPE": "1"}]'
python tools/time_big.py 4096 float64 exact 1 '[{}, {"CMG_ROWPAIR": "3", "CMG_RP_PIPE": "1"}]'
python tools/time_big.py 1024 float64 exact 1 '[{}, {"CMG_ROWPAIR": "3", "CMG_RP_PIPE": "1"}]'
