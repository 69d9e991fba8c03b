cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/b3.json 2> gpurun_out/b3.err; tail -2 gpurun_out/b3.err; cat gpurun_out/b3.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bref.json 2> gpurun_out/bref.err; tail -2 gpurun_out/bref.err; cat gpurun_out/bref.json
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/b4.json 2> gpurun_out/b4.err; tail -2 gpurun_out/b4.err; cat gpurun_out/b4.json
timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu > gpurun_out/b5.json 2> gpurun_out/b5.err; tail -2 gpurun_out/b5.err; cat gpurun_out/b5.json
