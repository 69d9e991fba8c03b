cd $GRAFT_REPO_ROOT
./tools/micro/tma_test3 4 116 95 95
./tools/micro/tma_test3 4 100 97 97
./tools/micro/tma_test3 4 116 94 95
./tools/micro/tma_test3 4 116 93 93
./tools/micro/tma_test3 8 68 95 95
./tools/micro/tma_test3 8 68 93 94
./tools/micro/tma_test3 4 36 1 1
./tools/micro/tma_test3 4 36 2 2
./tools/micro/tma_test3 4 36 4 4
