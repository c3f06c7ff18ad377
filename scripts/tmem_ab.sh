# tensor-memory accumulator groups (SGM_TM_FIRST=g: groups g..7 in TMEM, 8 = none) on the same build
for c in ${CFGS:-"1 64" "4 32"}; do set -- $c
for g in ${GS:-8 6 4 2}; do
echo "tm_first=$g $(SGM_TM_FIRST=$g python scripts/time_score.py --config $1 --views $2 --repeat 5 2>&1 | head -1)"
done; done
