#!/bin/bash
# SASS instruction count of each fused-kernel instantiation (code-size / I-cache budget)
for o in ${1:-build/obj}/dbp_kernel_n*.o; do
  n=$(cuobjdump -sass $o | grep -cE '^\s+/\*[0-9a-f]{4,5}\*/')
  echo "$(basename $o .o) $n instr ($((n*16/1024)) KB)"
done
