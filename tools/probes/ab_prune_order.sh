V=paper_2112_06300_b200/lib/variants/base/libccdk.so
for i in 1 2; do
  CCDK_LIB=$V python tools/ab.py step C4 10
  python tools/ab.py step C4 10
done
for w in C2 C3; do CCDK_LIB=$V python tools/ab.py step $w 10; python tools/ab.py step $w 10; done
CCDK_LIB=$V python tools/ab.py c5; python tools/ab.py c5
