# depth-prefix binning cap sweep on cfg4 (SGM_PREFIX_CAP): bash scripts/cap_sweep.sh <caps...>
python scripts/time_score.py --config 4 --views 32 --repeat 3 2>&1 | head -1
for c in ${@:-256 1024 4096 16384}; do echo cap $c; SGM_PREFIX_BINNING=1 SGM_PREFIX_CAP=$c python scripts/time_score.py --config 4 --views 32 --repeat 3 2>&1 | head -1; done
