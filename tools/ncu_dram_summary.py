import csv,collections,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
hdr=rows[0]
iid=hdr.index('ID'); im=hdr.index('Metric Name'); iv=hdr.index('Metric Value')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(int(r[iid]),{})[r[im]]=float(r[iv].replace(',',''))
names=sys.argv[2].split(',')
ids=sorted(d); per=len(ids)//len(names)
for k,nm in enumerate(names):
    grp=[d[i] for i in ids[k*per:(k+1)*per]]
    big=[g for g in grp if g['dram__bytes_read.sum']>1e9]
    g=big[-1]
    print(nm.ljust(28), {m.split('.')[0].replace('lts__t_sectors_srcunit_tex_op_','tex_'):round(v/1e6,1) for m,v in g.items()})
