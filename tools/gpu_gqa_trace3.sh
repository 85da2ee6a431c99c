ST_K1_TRACE_CTA=1 timeout 120 python tools/k1_trace.py gpurun_out/gq16.raw --B 16 --T 16 --H 64 --Hkv 8 --L 4096 --chain > gpurun_out/gq16_reg.txt 2>&1
ST_K1_TRACE_CTA=1 timeout 120 python tools/k1_trace.py gpurun_out/gq8.raw --B 16 --T 8 --H 64 --Hkv 8 --L 4096 --chain > gpurun_out/gq8_reg.txt 2>&1
