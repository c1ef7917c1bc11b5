for v in "$@"; do IL_LIB_VARIANT=$v timeout 300 python scripts/attn_trace.py > gpurun_out/trace_$v.txt 2>&1; echo $v=$?; done
