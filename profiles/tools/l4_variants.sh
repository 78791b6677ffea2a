#!/bin/bash
# A/B of the L >= 3 SIMT kernel variants (configs[3]); see DESIGN.md 3.x
V=paper_2601_16622_b200/_variants
cd "$(dirname "$0")/../.."
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fwd_bwd or bf16 or every_degree" > gpurun_out/l4_tests_A.log 2>&1; echo rc=$? >> gpurun_out/l4_tests_A.log
python bench.py --config 4 --no-cpu-baseline --no-gate --steps 5 > gpurun_out/l4_A.json 2>/dev/null
for x in B C D; do
  ES_LIB_PATH=$PWD/$V/$x.so python bench.py --config 4 --no-cpu-baseline --no-gate --steps 5 > gpurun_out/l4_$x.json 2>/dev/null
done
ES_LIB_PATH=$PWD/$V/B.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fwd_bwd or bf16" > gpurun_out/l4_tests_B.log 2>&1; echo rc=$? >> gpurun_out/l4_tests_B.log
