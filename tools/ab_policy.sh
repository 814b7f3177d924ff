for rep in 1 2; do
for v in default pol1 pol2; do
  if [ $v = default ]; then L=""; else L=paper_2112_06300_b200/lib/variants/$v/libccdk.so; fi
  for w in C4 C2; do CCDK_LIB=$L python tools/ab.py step $w 10 2>&1 | tail -1 | sed -e "s/^/$v /" | cut -c1-250; done
  CCDK_LIB=$L python tools/ab.py c5 10000000 2>&1 | tail -1 | sed -e "s/^/$v /"
done; done
