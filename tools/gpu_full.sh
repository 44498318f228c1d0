cd $GRAFT_REPO_ROOT
R=${R:-r8}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --depth ${DEPTH:-2} > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?" >> gpurun_out/${R}_bench.err
tail -n 15 gpurun_out/${R}_pytest.log; cat gpurun_out/${R}_bench.json; tail -n 20 gpurun_out/${R}_bench.err
