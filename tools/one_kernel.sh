#!/bin/bash
# Registers / stack / spill bytes of single kernel instances in seconds (no GPU):
#   tools/one_kernel.sh "stage_kernel<2, 144>(Tab, Phys, StageArgs)" ["-DQF_OCC2=4 ..."]
# compiles a translation unit that includes csrc/qf_kernels.cu without the C ABI
# (QF_KERNELS_ONLY) and explicitly instantiates the named __global__ templates
# (several, separated by ';').
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
{
  echo "#define QF_KERNELS_ONLY"
  echo "#include \"$ROOT/paper_1904_08684_b200/csrc/qf_kernels.cu\""
  echo "namespace qf {"
  IFS=';' read -ra KS <<< "$1"
  for k in "${KS[@]}"; do echo "template __global__ void $k;"; done
  echo "}"
} > $T/one.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr $2 \
     -Xptxas -v -cubin -o $T/one.cubin $T/one.cu 2>&1 | python3 -c "
import sys, re
t = sys.stdin.read()
for m in re.finditer(r'Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n.*?Used (\d+) registers', t, re.S):
    n = re.sub(r'_ZN2qf\d+', '', m.group(1)).split('EEEv')[0]
    if 'stage' in n or 'volume' in n or 'velocity' in n:
        print(f'{n:40s} regs {m.group(5):>4s} stack {m.group(2):>5s} spill st/ld {m.group(3)}/{m.group(4)}')
if 'error' in t: print(t[-3000:])
"
[ -n "$KEEP" ] && echo "cubin: $T/one.cubin" || rm -rf $T
