import sys,re,collections,json
def load(f):
    tot=collections.OrderedDict(); cnt=collections.Counter(); seq=[]
    for l in open(f):
        m=re.match(r'\s*([\d.]+) us\s+(.*)',l)
        if m:
            k=m.group(2).strip(); tot[k]=tot.get(k,0)+float(m.group(1)); cnt[k]+=1; seq.append((k,float(m.group(1))))
    return tot,cnt,seq
a=load(sys.argv[1]); b=load(sys.argv[2])
keys=list(dict.fromkeys(list(a[0])+list(b[0])))
for k in keys: print(f"{a[0].get(k,0):9.1f} {b[0].get(k,0):9.1f}  {k}")
print(f"{sum(a[0].values()):9.1f} {sum(b[0].values()):9.1f}  TOTAL")
for s in (a[2],b[2]):
    i=[n for n,(k,v) in enumerate(s) if 'colred_kernel<0>' in k]
    print([ (k[:24],v) for k,v in s[i[0]:i[0]+10]] if i else '')
