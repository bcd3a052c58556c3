for L in ${LIBS:-"" variants/batch.so}; do echo "== lib=${L:-default}"; env ${L:+LWB200_LIB=$L} timeout 600 python tools/bench_sweep.py --configs C2b,C2u,C3,C4 --no-cpu --reps 20 2>&1 | grep -i "work\|merge" | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: continue
    print(r['config'], r['matrix'][:30], r['dtype'], r['schedule'], r['ms'])
"; done
