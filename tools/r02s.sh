for b in 1 4 8; do for f in 0.35 0.5 0.65; do HETM_ZC_BLOCKS_PER_SM=$b HETM_ZC_FRACTION=$f timeout 300 python tools/e2e_probe.py | head -1 | python -c "
import sys,ast
l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):])
import statistics as st
tot=sum(st.median(v) for v in d.values())
print('zcb=$b zcf=$f', {k: round(st.median(v),2) for k,v in d.items()}, 'round_ms', round(tot,2))"; done; done
