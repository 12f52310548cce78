# latency-kernel phase trace (debug build): the NEXT=false (last) rotation is what stays in the buffer,
# so also trace with 12 rotations' worth by reading after one call
HEI_LIB_PATH=abl/lib_t.so timeout 300 python profiles/probes/w2_trace.py
