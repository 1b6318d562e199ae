"""Per-region instruction / stall-sample breakdown of an ncu source page (sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 24
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith('0x'):
        break
    data.append(r)
tot = sum(int(r[ix['Instructions Executed']]) for r in data)
samp = sum(int(r[ix['Warp Stall Sampling (All Samples)']]) for r in data)
print('total inst', tot, 'samples', samp, 'n', len(data))
for i in range(0, len(data), W):
    blk = data[i:i + W]
    inst = sum(int(r[ix['Instructions Executed']]) for r in blk)
    smp = sum(int(r[ix['Warp Stall Sampling (All Samples)']]) for r in blk)
    if inst > tot * 0.01 or smp > samp * 0.01:
        ops = ' '.join(sorted(set(r[1].split()[0] for r in blk if r[1].split() and not r[1].split()[0].startswith('@'))))[:100]
        print(data[i][0][-5:], str(inst).rjust(9), str(smp).rjust(5), ops)
