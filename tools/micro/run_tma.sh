cd $GRAFT_REPO_ROOT
for box in 36 68 72 100 116 128 200; do ./tools/micro/tma_test2 0 4 8 $box; done
./tools/micro/tma_test2 0 400 300 116
