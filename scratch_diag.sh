python scratch/diag3.py me 2>&1 | tail -4
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; grep '\[bench\]' gpurun_out/bench.err
