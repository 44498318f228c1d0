cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do SB_GSCFG=$v timeout 300 python tools/probe.py --n 512 --depths none --gs --gs-iters 100 2>&1 | tail -2 | sed "s/^/v$v /"; done
