# sustained bench: item-list schedule (default) vs regular k-blocks (SB_LIST=0,
# optionally SB_KBLK) in the experiment build, alternating
cd $GRAFT_REPO_ROOT
export SB200_LIB=$PWD/paper_1004_1741_b200/libsb200_exp.so
for rep in 1 2; do
  python bench.py --no-cpu --no-also --no-e2e > gpurun_out/listab_default_r${rep}.json 2>/dev/null
  SB_LIST=0 python bench.py --no-cpu --no-also --no-e2e > gpurun_out/listab_kblk_r${rep}.json 2>/dev/null
  SB_LIST=0 SB_KBLK=128 python bench.py --no-cpu --no-also --no-e2e > gpurun_out/listab_kb128_r${rep}.json 2>/dev/null
done
