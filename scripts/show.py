import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value %.0f %s  ms/step %.3f  matvec/s %.0f  e2e %.0f  launches %s" % (d["value"], d["unit"], d["ms_per_step"], d.get("matvec_per_s", 0), d["e2e"]["value"], d.get("gpu_launches")))
r = d["roofline"]; print("roofline", r["kernel"], "%.0f GB/s frac %.3f" % (r["achieved"], r["frac"]))
for k, v in d.get("stages", {}).items():
    print("  %-12s %8.1f us  %6.0f GB/s  share %.3f  n=%d" % (k, v["ms_per_launch"]*1e3, v["GBps"], v["share"], v["launches"]))
print("clocks", d.get("clocks"))
if len(sys.argv) > 2:
    for l in open(sys.argv[2]):
        d = json.loads(l); print(d['cfg'], d['prec'], 'setup %.2fs' % d['setup_s'], 'mv %.1fus' % (d['ms_per_matvec']*1e3), 'pt %.1fus' % (d['ms_per_freq_pt_profiled']*1e3), {k: d['stats'].get(k) for k in ('near_group_rows','near_row_order','near_union','nnz')})
        for k, v in d['stages'].items(): print('   %-12s %8.1f us %8.0f GB/s %8.1f MB' % (k, v['ms']*1e3, v['GBps'], v['MB']))
