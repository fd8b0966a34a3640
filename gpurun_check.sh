cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputest.log 2>&1; echo gputest rc=$?
tail -3 gpurun_out/r2c_gputest.log
timeout 600 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/r2c_bench.json
