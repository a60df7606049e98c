for m in rn18_224 rn50_224; do HSX_LIB_PATH=paper_2512_14628_b200/libhsx_trace.so python tools/k1_trace.py $m > gpurun_out/r2zn_k1trace_$m.txt 2>&1; done
head -12 gpurun_out/r2zn_k1trace_rn18_224.txt
