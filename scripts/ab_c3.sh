#!/bin/bash
python -m pytest tests/test_mfp_gpu.py -x -q -m gpu 2>&1 | tail -1
python scripts/tune_c3.py 32 32 64
