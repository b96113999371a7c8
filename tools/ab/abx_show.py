import json, glob, collections, statistics
d = collections.defaultdict(list)
for f in glob.glob('gpurun_out/abx_*.json'):
    n, c, r = f.split('/')[-1][4:-5].rsplit('_', 2)
    try:
        d[(n, c)].append(json.load(open(f))['value'])
    except Exception as e:
        d[(n, c)].append(float('nan'))
for k in sorted(d):
    print(k, [round(x) for x in d[k]], round(statistics.median(d[k])))
