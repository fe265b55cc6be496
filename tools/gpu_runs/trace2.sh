set -u
mkdir -p gpurun_out/trace2
IFA_B200_LIB=build/trc/libifa_b200.so timeout 200 python tools/pp_trace.py > gpurun_out/trace2/corr.txt 2>&1
IFA_B200_LIB=build/trd/libifa_b200.so timeout 200 python tools/pp_trace.py > gpurun_out/trace2/default.txt 2>&1
