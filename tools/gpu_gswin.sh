cd $GRAFT_REPO_ROOT
export SB200_LIB=$PWD/paper_1004_1741_b200/libsb200_exp.so
for rep in 1 2; do
for w in 2 3 4 6; do
  echo "window=$w rep=$rep" >> gpurun_out/gswin.log
  SB_GS_WINDOW=$w timeout 120 python tools/probe.py --n 512 --depths none --gs --gs-iters 100 >> gpurun_out/gswin.log 2>&1
done
done
