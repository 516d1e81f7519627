mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s1_tests.log 2>&1
python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
tail -3 gpurun_out/s1_tests.log; tail -c 1500 gpurun_out/s1_bench.json
