import re,sys,subprocess
lines=open(sys.argv[1]).read().splitlines()
cur=None; spill=''
pat=sys.argv[2] if len(sys.argv)>2 else ''
for l in lines:
    m=re.search(r"Compiling entry function '(\S+)'",l)
    if m: cur=m.group(1); spill=''
    if 'spill' in l: spill=l.strip()
    if 'registers' in l and cur:
        name=subprocess.run(['c++filt',cur],capture_output=True,text=True).stdout.strip()
        if pat in name: print(name[:60], l.split(':',1)[1].strip()[:40], '|', spill)
