for m in high low raster; do for c in "1 64" "4 32" "3 32"; do set -- $c; echo "prio=$m $(SGM_BIN_PRIO=$m python scripts/time_score.py --config $1 --views $2 --repeat 5 2>&1 | head -1)"; done; done
