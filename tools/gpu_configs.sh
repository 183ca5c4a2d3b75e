for c in cfg1 cfg3 cfg4; do
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  timeout 900 python bench.py --config $c --impl reference --steps 2 --warmup 1 > gpurun_out/cfg_${c}_ref.json 2> gpurun_out/cfg_${c}_ref.err
done
echo done
