for cv in "1.1,4" "1.05,2" "1.5,16"; do
tag=$(echo $cv | tr ',.' '__')
SUCO_TIE_CUT=$cv timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cut_${tag}_cfg4.json 2> /dev/null
SUCO_TIE_CUT=$cv timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cut_${tag}_cfg2.json 2> /dev/null
done
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cut_def_cfg4.json 2> /dev/null
echo done
