#!/bin/bash
# SASS digest of the hot kernels (cuobjdump -sass): instruction classes that
# show the TMA bulk copies (UBLKCP), mbarrier traffic (SYNCS), FP64 math and
# shared-memory loads.  The SG operator is JIT-compiled at setup: its C2 / C3
# sources are regenerated with tools/bin/sgop_src and compiled offline.
set -u
out=${1:-profiles/r02_sass_digest.txt}
lib=paper_2512_23027_b200/lib/libsgw_b200.so
tmp=$(mktemp -d)
count() {  # <sass file> <kernel label>
  printf "%-48s" "$2"
  for op in UBLKCP SYNCS DFMA DMUL DADD LDS LDG STG BAR.SYNC SHFL; do
    printf " %s=%d" "$op" "$(grep -cE "[[:space:]]$op" "$1")"
  done
  printf " total=%d\n" "$(grep -cE '^\s+/\*[0-9a-f]{4,}\*/' "$1")"
}
{
  echo "# SASS digest (cuobjdump -sass, sm_100a), $(date -u +%F)"
  cuobjdump -sass "$lib" > "$tmp/lib.sass"
  for k in pcg_fused_kernel pcg_phase_kernel walk_kernel "sweep_kernelILi2ELi12" "sweep_kernelILi1ELi24" sweep_generic_kernel; do
    awk -v k="$k" '/Function : /{p = index($0, k) > 0} p' "$tmp/lib.sass" > "$tmp/k.sass"
    [ -s "$tmp/k.sass" ] && count "$tmp/k.sass" "$k"
  done
  mkdir -p tools/bin
  nvcc -O2 -std=c++17 -x cu tools/sgop_src.cu paper_2512_23027_b200/csrc/host.cpp -o tools/bin/sgop_src -lnvrtc
  for c in "3 6 3 C2" "4 6 3 C3" "8 4 2 C5L8"; do
    set -- $c
    info=$(tools/bin/sgop_src $1 $2 $3 "$tmp/sg.cu")
    r=$(echo "$info" | grep -o "regs=[0-9]*" | cut -d= -f2)
    nvcc -cubin -arch=sm_100a -O3 -maxrregcount=$r "$tmp/sg.cu" -o "$tmp/sg.cubin" 2>/dev/null
    cuobjdump -sass "$tmp/sg.cubin" > "$tmp/sg.sass"
    count "$tmp/sg.sass" "sgop_kernel ($4: $info)"
  done
} > "$out"
rm -rf "$tmp"
cat "$out"
