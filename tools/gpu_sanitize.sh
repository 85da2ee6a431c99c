#!/bin/bash
# compute-sanitizer pass over the GPU parity tests (memcheck on every kernel
# family; racecheck + synccheck on the shared-memory kernels K2/K3/K4/masks).
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py tests/test_mss.py -q -k "not c2_shape" > $OUT/san.memcheck1.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_tc.py -q -k "matches_oracle or split or k_tree or gqa" > $OUT/san.memcheck2.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_kernels.py tests/test_mss.py -q -k "not c2_shape and not cuda_core" > $OUT/san.racecheck.txt 2>&1
timeout 1200 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_kernels.py tests/test_mss.py -q -k "not c2_shape and not cuda_core" > $OUT/san.synccheck.txt 2>&1
tail -n 2 $OUT/san.*.txt
