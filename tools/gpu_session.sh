cd $GRAFT_REPO_ROOT
for cfg in "64 4096" "256 4096" "1000 2048"; do for v in 0 5 6; do
  PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py $cfg 3
done; done
PCOTGPU_GS_PIPE_V=5 timeout 600 python -m pytest tests -m gpu -x -q -k "pipeline" 2>&1 | tail -2
