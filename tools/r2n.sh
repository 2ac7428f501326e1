bash tools/spacetime_sweep.sh
