set -x
python tools/golden_cfg5.py gpurun_out/cfg5_dmma.json > gpurun_out/golden.log 2>&1
mkdir -p tests/golden && cp gpurun_out/cfg5_dmma.json tests/golden/cfg5_dmma.json
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/b_cfg5.json 2> gpurun_out/b_cfg5.err
