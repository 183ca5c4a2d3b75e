COMM=1 timeout 600 python tools/prof_sharded.py > gpurun_out/prof_y1.log 2>&1
echo done
