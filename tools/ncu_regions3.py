import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
cur=None; res=[]
for r in rows:
    if r and r[0]=="File Path": cur=r[1].split("/")[-1]
    if len(r)>8 and r[0].isdigit() and r[2]=="-":
        res.append((cur,int(r[0]),int(r[7]),int(r[4]),r[1][:90]))
te=sum(x[2] for x in res); ts=sum(x[3] for x in res)
print("total warp instr",te,"samples",ts)
regions=[(47,81,"helpers"),(254,279,"mbar"),(290,308,"geom"),(309,322,"word1"),(324,403,"stage"),(405,424,"read/gv"),(426,460,"store_packed"),(462,508,"store"),(510,533,"pairfar/exhaust"),(535,550,"direct"),(577,579,"guess"),(601,635,"decode"),(646,730,"resolve"),(732,803,"unit setup"),(804,873,"pass1"),(874,905,"p2 words"),(906,927,"p2 warm"),(928,962,"p2 loop"),(963,1004,"p2 block"),(1005,1021,"p2 resolve+store"),(1023,1060,"kernel")]
agg=collections.Counter(); smp=collections.Counter()
for f,l,e,s,src in res:
    name=f
    if f=="k_sweep.cu":
        name="other"
        for a,b,n in regions:
            if a<=l<=b: name=n
    agg[name]+=e; smp[name]+=s
for k,v in agg.most_common(): print(f"{k:20s} {v/te*100:5.1f}% instr {smp[k]/ts*100:5.1f}% samples")
print("--- top lines by instr")
for f,l,e,s,src in sorted(res,key=lambda x:-x[2])[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    print(f"{e/te*100:5.1f}% {s/ts*100:5.1f}% {f}:{l} {src}")
