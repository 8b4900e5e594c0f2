#!/bin/bash
# A/B kernel-(a) variants on C3 (one process per env setting)
python -m pytest tests/test_mfp_gpu.py tests/test_e2_vs_reference.py -x -q -m gpu 2>&1 | tail -3
python scripts/tune_c3.py 32 64
DFX_TRACE=1 python scripts/one_solve.py 3 2>&1 | tail -14
