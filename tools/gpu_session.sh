cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "heat3d or s3d7 or golden or default_schedule or batch" 2>&1 | tail -2
timeout 300 python tools/kbench.py s3d7 --bts 1,2,3,4 --orders both 2>&1 | grep -E "GUpd"
