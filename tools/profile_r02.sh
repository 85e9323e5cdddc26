# Round-2 evidence run on one B200 (gpurun): bench lines for every config / mode, the N = 2
# spawn path (plumbing on one GPU), the reference arm, the ncu launch list and full captures of
# the j = 15 backward and forward launches.  Outputs under gpurun_out/r02_*.
set -x
P=${P:-gpurun_out/r02}    # output prefix
python bench.py > ${P}_bench_cfg3.json 2> ${P}_bench_cfg3.err
python bench.py --mode spaco --sampler paper --no-cpu-baseline > ${P}_bench_cfg3_spaco_paper.json 2>&1
python bench.py --mode spaco --sampler ht --no-cpu-baseline > ${P}_bench_cfg3_spaco_ht.json 2>&1
python bench.py --mode spaco --sampler bernoulli --no-cpu-baseline > ${P}_bench_cfg3_spaco_bernoulli.json 2>&1
python bench.py --deterministic --no-cpu-baseline > ${P}_bench_cfg3_det.json 2>&1
python bench.py --config cfg2 --no-cpu-baseline > ${P}_bench_cfg2.json 2>&1
python bench.py --config cfg5 --no-cpu-baseline > ${P}_bench_cfg5.json 2>&1
python bench.py --config cfg4 --steps 3 --no-cpu-baseline --no-e2e > ${P}_bench_cfg4.json 2>&1
python bench.py --config cfg1 --dtype fp32dbg --no-cpu-baseline > ${P}_bench_cfg1_fp32dbg.json 2>&1
python bench.py --config cfg2 --dtype fp32dbg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > ${P}_bench_cfg2_fp32dbg.json 2>&1
SECO_BENCH_SHARED_GPU=1 python bench.py --gpus 2 --config cfg2 --no-cpu-baseline --no-e2e > ${P}_bench_cfg2_gpus2_shared.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > ${P}_bench_reference.json 2>&1
python tools/launch_gaps.py cfg3 cfg3r8 cfg4r8 > ${P}_launch_gaps.txt 2>&1
python tools/kbench.py cfg3 0,1,3,7,15 10 > ${P}_kbench_cfg3.txt 2>&1
python tools/lora_bench.py > ${P}_lora_bench.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${P}_launches_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_ncu_launch.log 2>&1
python bench.py --profile-steps 2 > ${P}_ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:seco_bwd2_sm100 --launch-skip 16 --launch-count 1 \
    -o ${P}_bwd_j15 python bench.py --profile-steps 2 > ${P}_ncu_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:seco_fwd2?_sm100 --launch-skip 48 --launch-count 1 \
    -o ${P}_fwd_j15 python bench.py --profile-steps 2 > ${P}_ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lora -s 20 -c 2 -o ${P}_lora \
    python tools/lora_bench.py 2048 4096 4096 8 > ${P}_ncu_lora.log 2>&1
ls -la gpurun_out | grep r02
