set -x
python -m pytest tests/test_gpu_alloc.py -x -q 2>&1 | tail -5
BARGS="--no-cpu --no-parity --e2e-steps 0 --steps 2 --warmup 3"
python bench.py $BARGS > gpurun_out/b_small.json 2> gpurun_out/b_small.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02s3_launches_bench.csv python bench.py $BARGS > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ttmc3pq -s 3 -c 1 -f -o gpurun_out/r02s3_ttmc3 python bench.py --configs ttmc3 $BARGS > gpurun_out/ncu_t.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mttkrp3_smf -s 3 -c 1 -f -o gpurun_out/r02s3_mttkrp3_j python bench.py --configs mttkrp3_j $BARGS > gpurun_out/ncu_j.log 2>&1
ls -la gpurun_out/*.ncu-rep
