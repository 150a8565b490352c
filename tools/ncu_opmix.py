"""Executed-instruction mix (by SASS opcode) of the first launch of one kernel in an ncu report.

  python tools/ncu_opmix.py report.ncu-rep kernel_regex
"""
import csv, subprocess, sys, re, collections
rep, regex = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass','-k','regex:'+regex,'--launch-count','1'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
k0 = 1 if 'Source' in rows[1] else 0
h=rows[k0]; i_src=h.index('Source'); i_ie=h.index('Instructions Executed')
cnt=collections.Counter(); tot=0
for r in rows[k0+1:]:
    try: c=int(r[i_ie] or 0)
    except: continue
    src=r[i_src].strip()
    op=re.sub(r'^@!?U?P[T0-9]+\s+','',src).split(' ')[0]
    base=op.split('.')[0]
    cnt[base]+=c; tot+=c
for op,c in cnt.most_common(25): print(f"{op:12s} {c:>12d} {c/tot*100:5.1f}%")
print('total',tot)
