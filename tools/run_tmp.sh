cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_pcpg.py -q -x > gpurun_out/t_pcpg.log 2>&1
