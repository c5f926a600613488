# Bank-conflict model of k_mana_rowS block loads ("Next targets"):
# average wavefronts per LDS.128 phase over all digit shifts, for candidate 9-block layouts.
import itertools
D=5; NT=3**D
def digits(x):
    return [(x//3**j)%3 for j in range(D)]
def shifted(t,c,neg):
    td=digits(t); r=0
    for j in range(D):
        r+= (((6-td[j]-c[j])%3) if neg else ((td[j]-c[j]+3)%3))*3**j
    return r
layouts={
 'cur':lambda b:9*b,
 'skew8':lambda b:9*b+b//8,
 'skew3':lambda b:9*b+(b//3)%2,
 'skew9':lambda b:9*b+(b//9)%8,
 'pad10':lambda b:10*b,
 'skew27':lambda b:9*b+(b//3)%3,
 'skew_b9_4':lambda b:9*b+4*((b//9)%2),
}
import random
random.seed(1)
cs=[list(c) for c in itertools.product(range(3),repeat=D)]
for name,f in layouts.items():
    tot=0;n=0
    for c in cs:
        for neg in (0,1):
            for w in range(0,NT,32):
                for q in range(4):
                    ts=[t for t in range(w+8*q,min(w+8*q+8,NT))]
                    if not ts: continue
                    # k=0 instruction (all k similar shift)
                    groups={}
                    for t in ts:
                        b=shifted(t,c,neg); g=(f(b))%8
                        groups.setdefault(g,set()).add(b)
                    tot+=max(len(s) for s in groups.values()); n+=1
    print(name, tot/n)
