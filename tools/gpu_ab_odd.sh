# A/B of two library builds on the odd fused depths (T = 3, 1): $A vs $B
cd $GRAFT_REPO_ROOT
A=${A:-$PWD/paper_1004_1741_b200/libsb200.so}; B=${B:-$PWD/paper_1004_1741_b200/libsb200_prev.so}
OUT=gpurun_out/${R:-ab_odd}.log
for rep in 1 2 3; do
  for L in $A $B; do
    echo "lib=$(basename $L) rep=$rep" >> $OUT
    SB200_LIB=$L timeout 120 python tools/probe.py --n 1024 --iters 39 --depths 3,4 --reps 3 >> $OUT 2>&1
    SB200_LIB=$L timeout 120 python tools/probe.py --n 512 --iters 99 --depths 3,1 --reps 3 >> $OUT 2>&1
  done
done
