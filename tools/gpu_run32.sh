cd $GRAFT_REPO_ROOT
E='[{}, {"CMG_FUSE_MASK": "1", "CMG_TS2": "4", "CMG_TS3": "8"}, {"CMG_FUSE_MASK": "1", "CMG_TS2": "8", "CMG_TS3": "4"}, {"CMG_FUSE_MASK": "1", "CMG_TS2": "2", "CMG_TS3": "16"}]'
python tools/time_big.py 16384 float32 fast 1 "$E"
python tools/time_big.py 512 float32 fast 64 "$E"
python tools/time_big.py 1024 float64 exact 1 "$E"
python tools/time_big.py 1024 float32 fast 1 "$E"
python tools/time_big.py 1024 float64 fast 1 "$E"
