# A/B of two library builds on config 5's GS (512^3 x 100) and a 4-slab pipeline
cd $GRAFT_REPO_ROOT
A=${A:-$PWD/paper_1004_1741_b200/libsb200.so}; B=${B:-$PWD/paper_1004_1741_b200/libsb200_prev.so}
for rep in 1 2 3; do
  for L in $A $B; do
    echo "lib=$(basename $L) rep=$rep" >> gpurun_out/ab_gs.log
    SB200_LIB=$L timeout 120 python tools/probe.py --n 512 --depths none --gs --gs-iters 100 >> gpurun_out/ab_gs.log 2>&1
  done
done
