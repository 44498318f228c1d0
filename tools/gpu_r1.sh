cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 300 python tools/probe.py --n 512 --iters 8 --depths 1,2,4,8 > gpurun_out/r1_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/r1_probe.log
timeout 300 python tools/probe.py --n 256 --iters 8 --depths 1 --gs --gs-iters 2 > gpurun_out/r1_probe_gs.log 2>&1; echo "probe gs rc=$?" >> gpurun_out/r1_probe_gs.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
tail -5 gpurun_out/r1_*.log
