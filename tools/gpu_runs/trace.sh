set -u
mkdir -p gpurun_out/trace
IFA_B200_LIB=build/pptrace/libifa_b200.so timeout 300 python tools/pp_trace.py > gpurun_out/trace/pp_trace_launder.txt 2>&1
