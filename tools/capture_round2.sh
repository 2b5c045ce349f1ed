# Round-end capture, part 2 (development tool): ncu --set full of the fused partition sort and
# of the scheduler's cooperative re-key + pop kernel.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"part_fused" --launch-skip 4 -c 1 -o gpurun_out/prof_rank_r01p python tools/kernel_ab.py > gpurun_out/ncu_rank_r01p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rekey_pop_seq" --launch-skip 20 -c 1 -o gpurun_out/prof_rekey_r01p python -c "
import bench_sched, paper_2604_00499_b200 as tie
bench_sched.run(tie, tie.McContext(3.5), sizes=(1000000,), variants=('rekey',), cpu=False, steps=30)" > gpurun_out/ncu_rekey_r01p.log 2>&1
