#!/bin/bash
# SASS census of a variant .so: instruction counts of the production kernels' bodies and of the
# serial engine's out-of-line functions, plus the uniform-datapath opcodes in se::w32 (a w32 of
# ~560 instructions with ~19 UISETP and no R2UR is the fast form; see profiles/r02/ab_uniform.txt)
# usage: bash tools/sass_census.sh variants/x.so
set -e
T=$(mktemp -d); cd $T; cuobjdump -xelf all "$OLDPWD/$1" >/dev/null 2>&1
nvdisasm -c polarsc.sm_100a.cubin > all.dis 2>/dev/null
for K in ILi3ELb0ELb0ELi256ELi0E ILi3ELb1ELb0ELi512ELi4E ILi3ELb1ELb0ELi512ELi0E; do
  awk -v K=$K '/^\$?_Z[^ ]*:$/ {if (name!="") print n, name; name=$1; n=0} /^ +\/\*[0-9a-f]+\*\//{n++} END{print n,name}' all.dis \
    | grep $K | sed 's/_Z16sc_decode_kernel//; s/EEv9DecParams//g' | awk '{printf "%s=%s  ", $2, $1}'; echo
  awk -v K=$K 'BEGIN{on=0} /^\$?_Z[^ ]*:$/ {on = index($1, "_ZN2se3w32Eij")>0 && index($1,K)>0} on && /^ +\/\*[0-9a-f]+\*\//{print}' all.dis \
    | grep -oE "\b(R2UR|UISETP|BSSY|WARPSYNC|USEL|UIADD3|ULOP3|UMOV|BRA\.DIV)\b" | sort | uniq -c | tr '\n' ' '; echo
done
rm -rf $T
