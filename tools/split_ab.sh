#!/bin/bash
# Split lane copies (DOS_H2D_SPLIT / DOS_D2H_SPLIT): engine tests with the
# split on, then the 7B phase A/B alternated on one box
mkdir -p gpurun_out
DOS_H2D_SPLIT=3 DOS_D2H_SPLIT=2 timeout 900 python -m pytest tests/test_gpu_execute.py tests/test_gpu_engine_random.py -m gpu -x -q > gpurun_out/split_tests.txt 2>&1
echo "split tests rc=$? $(tail -1 gpurun_out/split_tests.txt)"
timeout 2400 bash tools/env_ab.sh split_ab - "DOS_H2D_SPLIT=2" "DOS_H2D_SPLIT=4" "DOS_H2D_SPLIT=2 DOS_D2H_SPLIT=2" - "DOS_H2D_SPLIT=2" "DOS_H2D_SPLIT=4" "DOS_H2D_SPLIT=2 DOS_D2H_SPLIT=2"
