cd $GRAFT_REPO_ROOT
R=${R:-r5}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${R}_smoke.log
timeout 300 python tools/probe.py --n 512 --iters 8 --depths 1,2,4,8 > gpurun_out/${R}_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/${R}_probe.log
timeout 300 python tools/probe.py --n 256 --iters 8 --depths 1 --gs --gs-iters 2 > gpurun_out/${R}_probe_gs.log 2>&1; echo "probe gs rc=$?" >> gpurun_out/${R}_probe_gs.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest.log
for f in gpurun_out/${R}_*.log; do echo "== $f"; tail -n 12 $f; done
