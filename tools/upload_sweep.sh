# scene-upload staging A/B inside bench.py's e2e (CCDK_STAGE_NT / _THREADS / _CHUNK_KB), interleaved
for rep in 1 2; do
for cfg in "0 7 2048" "1 7 2048" "1 7 1024" "1 3 2048" "1 3 1024"; do set -- $cfg
 CCDK_STAGE_NT=$1 CCDK_STAGE_THREADS=$2 CCDK_STAGE_CHUNK_KB=$3 python bench.py --steps 30 --warmup 3 --c5-queries 100000 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err
 python -c "
import json, statistics as st; d=json.load(open('/tmp/b.json')); s=d['e2e']['steps_ms']
print('nt $1 helpers<=$2 chunk $3: device', round(d['value'],3), 'e2e mean', round(st.mean(s),3), 'median', round(st.median(s),3), 'min', min(s), 'max', max(s))"
done; done
