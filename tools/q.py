import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d["ms_per_step"], {k: round(v,4) for k,v in d["stage_seconds"].items()}, round(d["roofline"]["frac"],4), d.get("parity"))
