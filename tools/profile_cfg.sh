# ncu evidence for one config (run on the B200 box from the repo root):
#   bash tools/profile_cfg.sh cfg4 r02
# 1. per-launch time + DRAM bytes of one query step's kernels (clock-control none);
# 2. one `--set full` capture each of the select, re-rank and traversal kernels of a query step
#    and of the k-means assignment kernel of the index build (source-correlated, -lineinfo).
set -u
CFG=$1; TAG=$2
B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 0 --config $CFG"
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"^(dense_(hist|fused|emit|plan|bound|compact|flag)|rerank|traverse|rank_halves|topk|select|shard|merge)" \
  --csv --log-file $O/${TAG}_${CFG}_launches.csv $B > /dev/null 2>&1
echo "launches rc=$?"
for K in "dense_fused" "rerank_(screen|u8_pipe|q8)" "traverse_thread" "rank_halves" "dense_compact_kernel" "assign_kernel"; do
  N=$(echo "$K" | tr -cd 'a-z_')
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 \
    -o $O/${TAG}_${CFG}_${N} $B > /dev/null 2>&1
  echo "$K rc=$?"
done
