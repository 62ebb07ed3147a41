import json, sys
for f in sys.argv[1:]:
    for ln in open(f):
        if ln.startswith('{'):
            d = json.loads(ln)
            print("%-28s %10.0f ins/s  ms/step %8.2f  K1 ms %8.2f  frac %.3f  e2e %10.0f  recall %s" % (
                f.split('/')[-1], d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline']['frac'],
                d['e2e']['value'], d.get('recall_at_k')))
