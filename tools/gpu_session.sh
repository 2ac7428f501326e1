cd $GRAFT_REPO_ROOT
for r in 1 2 3; do for v in 1 0; do PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 128 4000 2; done; done
for cfg in "13 4000" "25 1000" "100 2000" "64 4096"; do for v in 1 0 2; do
  PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py $cfg 2
done; done
timeout 600 python -m pytest tests -m gpu -x -q -k "gs" 2>&1 | tail -3
