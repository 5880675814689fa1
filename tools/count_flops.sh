#!/bin/bash
# Flops per pair interaction of the compiled direct kernels, from their SASS:
# FFMA = 2, FMUL / FADD = 1 (per pair = per MUFU.RSQ).  Used for flops_per_pair (fmm.cu)
# and bench.py's P2P figure.
obj=${1:-paper_1612_04082_b200/build/direct.o}
for k in "ILb1ELb0ELb0 U" "ILb0ELb1ELb0 P" "ILb1ELb1ELb0 UP" "ILb1ELb0ELb1 D" "ILb0ELb1ELb1 S" "ILb1ELb1ELb1 DS"; do
  set -- $k
  cuobjdump -sass "$obj" | awk -v K="direct_kernel$1" '$0 ~ "Function : .*"K {f=1; next} f && /Function : / {f=0} f' \
    | grep -E "^\s+/\*[0-9a-f]+\*/" | awk -v name=$2 '
      /MUFU.RSQ/ {n++} / FFMA(\.FTZ)? / {ffma++} / FMUL(\.FTZ)? / {fmul++} / FADD(\.FTZ)? / {fadd++}
      END {printf "%-3s pairs %d  flops/pair %.1f\n", name, n, (2*ffma+fmul+fadd)/n}'
done
