# geometry-fill A/B: points per thread of the alpha-from-geometry kernel
for ppt in ${PPTS:-1 2 4 11}; do P2S_GEO_PPT=$ppt python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ppt $ppt geometry', round(d['geometry_fill']['value']), 'resident', round(d['value']))"; done
