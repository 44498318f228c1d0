cd $GRAFT_REPO_ROOT
R=${R:-r8}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --depth 4 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?" >> gpurun_out/${R}_bench.err
timeout 900 python bench.py --steps 3 --warmup 3 --depth 3 --no-also --no-e2e --no-cpu > gpurun_out/${R}_bench_d3.json 2> gpurun_out/${R}_bench_d3.err
tail -n 3 gpurun_out/${R}_pytest.log; tail -n 3 gpurun_out/${R}_bench.err
