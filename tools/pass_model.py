from paper_1802_08032_b200 import circuits as C
c = C.layered_random_circuit(30, 20, 12345)
ops=[]
for o in c.ops:
    m=o.m8(); diag = m[2]==0 and m[3]==0 and m[4]==0 and m[5]==0
    ops.append((o.name, o.target, o.controls, diag))
H=5970; F=2500; T=2000; CREG=550; CLANE=1200; CSEL=650; COUT=300
def simulate(maxt, maxp):
    passes=[]; cur=None
    def new():
        return dict(tile=[], phases=[[]], ops=[])
    cur=new()
    def place(p, op):
        name,t,ctr,diag=op
        if not diag and t>=3:
            ph=p['phases'][-1]
            if t<5:
                if t not in ph and len(ph)<3: ph.append(t)
            else:
                if t not in p['tile'] and len(p['tile'])>=maxt: return False
                if t not in ph and len(ph)>=3:
                    if len(p['phases'])>=maxp: return False
                    p['phases'].append([])
                if t not in p['phases'][-1]: p['phases'][-1].append(t)
                if t not in p['tile']: p['tile'].append(t)
        p['ops'].append((op, len(p['phases'])-1))
        return True
    for op in ops:
        if not place(cur, op):
            passes.append(cur); cur=new(); place(cur, op)
        if len(cur['ops'])>=63: passes.append(cur); cur=new()
    passes.append(cur)
    tot=0
    for p in passes:
        tile=set(range(5))|set(p['tile'])
        comp=F+T*(len(p['phases'])-1)
        for (op,ph) in p['ops']:
            name,t,ctr,diag=op
            regs=p['phases'][ph]
            outer = any(cq not in tile for cq in ctr)
            if outer: comp+=COUT; continue
            if not diag and (t<3 or (t<5 and t not in regs)): comp+=CLANE
            elif ctr: comp+=CSEL
            else: comp+=CREG
        tot+=max(H,comp)
    return len(passes), tot
for mt,mp,meas in [(7,8,12.87*66),(7,2,10.19*80.67),(7,1,5.87*161.3),(6,8,10.70*77.7),(5,8,9.15*93)]:
    n,tot=simulate(mt,mp)
    print(mt,mp,n, "pred ms/step %.0f"%(tot*1771/1.965e6), "meas %.0f"%meas)

def dp(maxp=8):
    n=len(ops); INF=1e18; best=[INF]*(n+1); best[0]=0; cut=[0]*(n+1)
    for i in range(n):
        if best[i]>=INF: continue
        p=dict(tile=[], phases=[[]], ops=[]); comp=F
        for j in range(i, min(n, i+63)):
            op=ops[j]; name,t,ctr,diag=op
            # place
            ok=True
            if not diag and t>=3:
                ph=p['phases'][-1]
                if t<5:
                    if t not in ph and len(ph)<3: ph.append(t)
                else:
                    if t not in p['tile'] and len(p['tile'])>=7: ok=False
                    elif t not in ph and len(ph)>=3:
                        if len(p['phases'])>=maxp: ok=False
                        else: p['phases'].append([]); comp+=T
                    if ok:
                        if t not in p['phases'][-1]: p['phases'][-1].append(t)
                        if t not in p['tile']: p['tile'].append(t)
            if not ok: break
            tile=set(range(5))|set(p['tile'])
            regs=p['phases'][-1]
            outer = any(cq not in tile for cq in ctr)
            # note: outer-ness can change as tile grows; approximate with current tile
            if outer: comp+=COUT
            elif not diag and (t<3 or (t<5 and t not in regs)): comp+=CLANE
            elif ctr: comp+=CSEL
            else: comp+=CREG
            c=best[i]+max(H,comp)
            if c<best[j+1]: best[j+1]=c; cut[j+1]=i
    k=n; np_=0
    while k>0: k=cut[k]; np_+=1
    return np_, best[n]
n,tot=dp()
print("DP", n, "pred ms/step %.0f"%(tot*1771/1.965e6))
