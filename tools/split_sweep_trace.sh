for sp in "0,0,0,0" "4,0,0,0" "3,0,0,0" "12,0,0,0" "0,6,0,0" "0,4,0,0" "0,0,6,0" "0,0,3,0" "0,0,2,0" "0,0,0,12" "0,0,0,8" "0,0,0,6"; do
  r=$(TF_SPLITS=$sp TF_TRACE=1 TRACE_REPS=6 python tools/trace_step.py c2 0 2>&1 | grep -A6 "mean over" | tr '\n' ' ' | sed 's/  */ /g')
  echo "$sp | $r" | python -c "
import sys,re
l=sys.stdin.read(); sp=l.split('|')[0].strip()
step=re.search(r'step ([0-9.]+) us',l).group(1)
ks=re.findall(r'(\w+) mean incr ([0-9.]+) us',l)
print(sp, step, ' '.join(f'{k}={v}' for k,v in ks))"
done
