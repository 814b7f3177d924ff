# Interleaved A/B of tools/build_variant.py builds: bash tools/ab_variants.sh name1 name2 ...
# ("default" = the in-tree build; "env:VAR=VALUE" = the in-tree build under an environment switch);
# device-resident C4/C2/C3 steps and the C5 narrow batch.
for rep in 1 2; do
for v in "$@"; do
  E="CCDK_AB=1"
  if [ "$v" = default ]; then L=""; elif [[ "$v" == env:* ]]; then L=""; E="${v#env:}"; else L=paper_2112_06300_b200/lib/variants/$v/libccdk.so; fi
  for w in C4 C2 C3; do
    env $E CCDK_LIB=$L python tools/ab.py step $w 10 2>&1 | tail -1 | python -c "
import sys, ast; l=sys.stdin.read().strip(); d=ast.literal_eval(l[l.index('{'):]); print('$v', '$w', 'narrow', d['ms_narrow'], 'total', d['ms_total'], l.split(' toi ')[1].split(' ')[0])"
  done
  env $E CCDK_LIB=$L python tools/ab.py c5 10000000 2>&1 | tail -1 | sed -e "s/^/$v /"
done; done
