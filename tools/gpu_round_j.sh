B="timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3"
for t in 1 2 4 8; do SUCO_TILES=$t $B > gpurun_out/j_t$t.json 2>/dev/null; done
echo done
