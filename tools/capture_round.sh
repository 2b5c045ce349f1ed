# Round-end capture (development tool): GPU tests, bench, reference arm, ncu launch list and
# ncu --set full captures of the main kernels.  Run from the repo root on a B200 box.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r01p.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_r01p.json 2> gpurun_out/bench_r01p.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01p.json 2> gpurun_out/bench_ref_r01p.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01p.csv python bench.py --steps 2 --warmup 1 > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"score_coop|part_fused" --launch-skip 6 -c 2 -o gpurun_out/prof_r01p python tools/kernel_ab.py > gpurun_out/ncu_r01p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fit_lanes" -c 1 -o gpurun_out/prof_fit_r01p python tools/fit_probe2.py > gpurun_out/ncu_fit_r01p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rekey_pop_seq|step_apply" --launch-skip 40 -c 2 -o gpurun_out/prof_sched_r01p python bench_sched.py 1000000 > gpurun_out/ncu_sched_r01p.log 2>&1
