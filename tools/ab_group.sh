# A/B of group-mapped warp-kernel variants over the sweep matrices (fp32 + fp64)
for L in ${LIBS:-DEFAULT}; do echo "== lib=$L"; [ "$L" = DEFAULT ] && L=; env ${L:+LWB200_LIB=$L} timeout 600 python tools/bench_sweep.py --configs ${CONFIGS:-C2b,C2u,C3,C4} --no-cpu --reps 20 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: continue
    if r['schedule'] in ('${SCHED:-group_warp}',): print(r['config'], r['matrix'][:48], r['dtype'], r['schedule'], r['ms'])
"; done
