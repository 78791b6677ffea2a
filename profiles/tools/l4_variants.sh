#!/bin/bash
# A/B of the L >= 3 SIMT kernel variants (configs[3]; DESIGN.md 3.7,
# profiles/r02e_l4_variants.jsonl).
#
# Build the variants here first (nvcc cross-compiles; each is a full library):
#   V=paper_2601_16622_b200/_variants
#   ES_NVCC_EXTRA="-DES_L34_FWD_CPL=1" ES_LIB_OUT=$PWD/$V/B.so python -m paper_2601_16622_b200.build
#   ES_NVCC_EXTRA="-DES_L34_FWD_CPL=1 -DES_L34_BLK=0" ES_LIB_OUT=$PWD/$V/C.so python -m paper_2601_16622_b200.build
#   ES_NVCC_EXTRA="-DES_L34_FWD_CPL=1 -DES_L34_BLK=0 -DES_L34_QSMEM=0 -DES_L34_QRELOAD=0" \
#       ES_LIB_OUT=$PWD/$V/D.so python -m paper_2601_16622_b200.build
# then on the B200:  gpurun -- 'bash profiles/tools/l4_variants.sh'
V=paper_2601_16622_b200/_variants
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fwd_bwd or bf16 or every_degree" > gpurun_out/l4_tests_A.log 2>&1; echo rc=$? >> gpurun_out/l4_tests_A.log
python bench.py --config 4 --no-cpu-baseline --no-gate --steps 5 > gpurun_out/l4_A.json 2>/dev/null
for x in B C D; do
  [ -f $V/$x.so ] || continue
  ES_LIB_PATH=$PWD/$V/$x.so python bench.py --config 4 --no-cpu-baseline --no-gate --steps 5 > gpurun_out/l4_$x.json 2>/dev/null
  ES_LIB_PATH=$PWD/$V/$x.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fwd_bwd or bf16" > gpurun_out/l4_tests_$x.log 2>&1; echo rc=$? >> gpurun_out/l4_tests_$x.log
done
