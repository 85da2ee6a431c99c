timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_mss.py -q > gpurun_out/san.racecheck_k4.txt 2>&1; tail -2 gpurun_out/san.racecheck_k4.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_mss.py -q > gpurun_out/san.memcheck_k4.txt 2>&1; tail -2 gpurun_out/san.memcheck_k4.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_mss.py -q > gpurun_out/san.synccheck_k4.txt 2>&1; tail -2 gpurun_out/san.synccheck_k4.txt
python tools/mss_bench.py
