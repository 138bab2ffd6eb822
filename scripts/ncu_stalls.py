import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
col={h:i for i,h in enumerate(hdr)}
stalls=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot={s:0 for s in stalls}
S=0
def f(x):
    try: return float(x)
    except: return 0.0
data=[r for r in data if len(r)>=len(hdr)]
for r in data:
    S+=f(r[col['# Samples']])
    for s in stalls: tot[s]+=f(r[col[s]])
print('total samples',S, 'instr', sum(f(r[col['Instructions Executed']]) for r in data))
for s,v in sorted(tot.items(), key=lambda kv:-kv[1])[:12]: print(f'{s:28s} {v:9.0f} {100*v/S:5.1f}%')
top=sorted(data,key=lambda r:-f(r[col['# Samples']]))[:int(sys.argv[2]) if len(sys.argv)>2 else 40]
for r in top:
    ss=sorted(((f(r[col[s]]),s) for s in stalls),reverse=True)[:2]
    print(r[col['Address']][-5:], f"{f(r[col['# Samples']]):7.0f}", f"{f(r[col['Instructions Executed']]):9.0f}", r[col['Source']][:70], ss)
