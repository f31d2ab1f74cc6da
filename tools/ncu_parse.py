"""Aggregate an ncu launch list CSV by kernel name, grid and block size: launches and serialised time. usage: python tools/ncu_parse.py launches.csv [top]"""
import csv,collections,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ii=h.index("ID")
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii],{})["name"]=r[ki]; d[r[ii]][r[mi]]=r[vi]
agg=collections.defaultdict(lambda:[0,0.0])
for k,v in d.items():
    nm=v["name"].split("(")[0][-40:]; key=(nm,v.get("launch__grid_size"),v.get("launch__block_size"))
    agg[key][0]+=1; agg[key][1]+=float(v.get("gpu__time_duration.sum","0").replace(",",""))
for k,(n,t) in sorted(agg.items(), key=lambda kv:-kv[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    print(f"{t/1e6:8.3f} ms  n={n:4d}  {k}")
