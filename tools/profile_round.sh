set -x
python bench.py > gpurun_out/r01d_bench_cfg3.json 2> gpurun_out/r01d_bench_cfg3.err
python bench.py --config cfg3 --mode spaco --no-cpu-baseline > gpurun_out/r01d_bench_cfg3_spaco.json 2>&1
python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/r01d_bench_cfg2.json 2>&1
python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/r01d_bench_cfg5.json 2>&1
python bench.py --config cfg4 --steps 3 --no-cpu-baseline > gpurun_out/r01d_bench_cfg4.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01d_bench_reference.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01d_launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:seco_bwd2_sm100 --launch-skip 16 --launch-count 1 -o gpurun_out/r01d_bwd_j15 python bench.py --profile-steps 2 > gpurun_out/ncu_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:seco_fwd_sm100 --launch-skip 48 --launch-count 1 -o gpurun_out/r01d_fwd_j15 python bench.py --profile-steps 2 > gpurun_out/ncu_fwd.log 2>&1
ls -la gpurun_out
