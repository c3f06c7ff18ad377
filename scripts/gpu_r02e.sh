for c in 1 4; do n=8; [ $c = 4 ] && n=4
python scripts/profile_raster.py --config $c --views $n > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launch_cfg$c.csv python scripts/profile_raster.py --config $c --views $n --repeat 2 > /dev/null 2>&1; echo ncu$c=$?
done
for c in 1 3 4; do n=64; [ $c = 4 ] && n=32; [ $c = 3 ] && n=32; timeout 600 python scripts/time_score.py --config $c --views $n --repeat 3 2>&1 | head -1; done
