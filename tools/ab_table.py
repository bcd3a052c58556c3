import sys,re,collections
cur=None; tab=collections.OrderedDict(); libs=[]
for l in sys.stdin:
    l=l.rstrip()
    if l.startswith('== lib='): cur=l[7:]; libs.append(cur); continue
    m=re.match(r'(C\S+) (.*) (float\d\d) (\S+) ([\d.]+)$',l)
    if m and cur:
        k=(m.group(1)+' '+m.group(2)[:22]+' '+m.group(3)); tab.setdefault(k,{})
        kk=k; i=2
        while cur in tab[kk]: kk=k+'#'+str(i); tab.setdefault(kk,{}); i+=1
        tab[kk][cur]=m.group(5)
    elif not m: print(l)
print(' '*36+' '.join(f'{x.split("/")[-1][:9]:>9s}' for x in libs))
for k,v in tab.items(): print(f'{k:36s}'+' '.join(f'{v.get(x,"-"):>9s}' for x in libs))
