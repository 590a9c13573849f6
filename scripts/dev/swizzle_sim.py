# simulate smem bank conflicts of the row-pass exchange for padded vs xor-swizzled layouts
def bitrev(q,R):
    r=0;b=1
    while b<R: r=(r<<1)|(q&1); q>>=1; b<<=1
    return r
def plan(S_LOG,E_LOG=5):
    Q=(S_LOG+E_LOG-1)//E_LOG
    rl=[E_LOG if r<Q-1 else S_LOG-E_LOG*(Q-1) for r in range(Q)]
    gl=[sum(rl[:r]) for r in range(Q)]
    return Q,rl,gl
def sim(S_LOG, layout, V):
    S=1<<S_LOG; E=32; TPV=S//E; Q,rl,gl=plan(S_LOG)
    threads=V*TPV
    RS=S+S//32
    def phys(w,p):
        if layout=='pad': return w*RS+p+(p>>5)
        P=w*S+p
        return P ^ ((P>>5)&31)
    worst={}
    # writes of round rho (rho<Q-1), reads of round rho>=1
    for rho in range(Q):
        R=1<<rl[rho]; G=1<<gl[rho]; T=S//(G*R); NG=E//R
        if rho>=1:
            # reads: x[h*R+m] = sm[q + (S/R)*m], q=v+TPV*h
            for h in range(NG):
                for m in range(R):
                    for warp in range(threads//32):
                        banks={}
                        for lane in range(32):
                            t=warp*32+lane; w=t//TPV; v=t%TPV
                            q=v+TPV*h
                            a=phys(w,q+(S//R)*m)
                            banks.setdefault(a%32,set()).add(a)
                        c=max(len(s) for s in banks.values())
                        worst[('rd',rho)]=max(worst.get(('rd',rho),1),c)
        if rho<Q-1:
            for h in range(NG):
                for mm in range(R):
                    for warp in range(threads//32):
                        banks={}
                        for lane in range(32):
                            t=warp*32+lane; w=t//TPV; v=t%TPV
                            q=v+TPV*h; g=q%G; tt=q//G; k=bitrev(mm,R)
                            if rho==0: pos=k+R*tt
                            else: pos=g+G*k+G*R*tt
                            a=phys(w,pos)
                            banks.setdefault(a%32,set()).add(a)
                        c=max(len(s) for s in banks.values())
                        worst[('wr',rho)]=max(worst.get(('wr',rho),1),c)
    return worst
for S_LOG in range(6,15):
    V=max(1,min(2048>>S_LOG, 1<<(S_LOG-1))) if S_LOG<11 else 1
    print(S_LOG, V, 'pad', sim(S_LOG,'pad',V), 'xor', sim(S_LOG,'xor',V))
