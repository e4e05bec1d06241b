for ex in "birth_cov=0.25,0.25,1.0,0.1,0.1" "birth_cov=1.0,1.0,1.0,0.1,0.1" "birth_cov=4.0,4.0,4.0,0.3,0.1" "sigma_a=1.0;sigma_w=0.5" "sigma_a=1.0;sigma_w=0.5;birth_cov=1.0,1.0,1.0,0.1,0.1"; do
 for nh in "20 100" "10 25"; do
  timeout 300 python profiles/convoy_seeds.py $nh 0,1,2,3,4,5,6,7,8,9 "$ex" | python -c "
import sys, json, numpy as np
L=[json.loads(l) for l in sys.stdin if l.startswith('{')]
c=np.array([d['card_err'] for d in L]); t=np.array([d['track_err_m'] for d in L])
print('$ex', '$nh', round(c.mean(),4), round(c.std(ddof=1)/np.sqrt(len(c)),4), round(t.mean(),4), [round(x,3) for x in c])"
 done
done
