cd $GRAFT_REPO_ROOT
for it in 1 2 4 8 16 32; do for v in 0 1; do
SB_GSCFG=$v timeout 120 python tools/probe.py --n 512 --depths none --gs --gs-iters $it 2>&1 | grep naive | sed -E 's/"roof1_frac.*//' | sed "s/^/it=$it v=$v /"
done; done
