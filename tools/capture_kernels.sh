# ncu --set full captures of the score, fused rank and scheduler kernels (development tool).
#   bash tools/capture_kernels.sh <tag>      (on the GPU box, from the repo root)
# Reports land in gpurun_out/prof_{score,rank,sched}_<tag>.ncu-rep; read them here with
# ncu -i ... --page raw --csv / --page source --csv, summaries go to profiles/.
tag=${1:-dev}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"score_coop" --launch-skip 6 -c 1 -o gpurun_out/prof_score_$tag python tools/kernel_ab.py > gpurun_out/ncu_score_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"part_fused" --launch-skip 4 -c 1 -o gpurun_out/prof_rank_$tag python tools/kernel_ab.py > gpurun_out/ncu_rank_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"step_apply" --launch-skip 40 -c 1 -o gpurun_out/prof_sched_$tag python -c "
import bench_sched, paper_2604_00499_b200 as tie
bench_sched.run(tie, tie.McContext(3.5), sizes=(67108864,), variants=('steady',), cpu=False, steps=30)" > gpurun_out/ncu_sched_$tag.log 2>&1
