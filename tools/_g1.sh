set -x
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; free -g > gpurun_out/free.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg5.json 2> gpurun_out/b_cfg5.err
PPC_OZAKI=0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg5_dmma.json 2> gpurun_out/b_cfg5_dmma.err
python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err
python bench.py --workload cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
