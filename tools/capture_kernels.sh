# ncu captures of the path's kernels (development tool):
#   bash tools/capture_kernels.sh <tag>      (on the GPU box, from the repo root)
# --set full of the score kernel, the fused rank kernel (config 2, 1M), the fit kernel
# (config 3, 1M x 16) and the level-2 partition sort (config 4, 64M), plus the launch list of a
# short bench run.  Reports land in gpurun_out/; read them here with tools/ncu_summary.py and
# tools/make_traffic.py, summaries go to profiles/.
tag=${1:-dev}
mkdir -p gpurun_out
full="ncu --set full --clock-control none --import-source on"
timeout 600 $full -k regex:"score_coop" --launch-skip 6 -c 1 -o gpurun_out/prof_score_$tag python tools/kernel_ab.py > gpurun_out/ncu_score_$tag.log 2>&1
timeout 600 $full -k regex:"part_fused" --launch-skip 4 -c 1 -o gpurun_out/prof_rank_$tag python tools/kernel_ab.py > gpurun_out/ncu_rank_$tag.log 2>&1
timeout 600 $full -k regex:"fit_lanes" -c 1 -o gpurun_out/prof_fit_$tag python tools/fit_probe2.py > gpurun_out/ncu_fit_$tag.log 2>&1
timeout 600 $full -k regex:"part_l2" --launch-skip 2 -c 1 -o gpurun_out/prof_l2_$tag python tools/rank64_probe.py > gpurun_out/ncu_l2_$tag.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/bench_under_ncu_$tag.log 2>&1
