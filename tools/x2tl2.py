import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'x2_timeline.py')).read().split("d = np.diff")[0])
names = {0:"start",2:"init sync",3:"Bfr stored",5:"window arrived",1:"after Bfr sync (phi0 start)",4:"phi1 start",6:"contract1 end",7:"end"}
for k in [2,3,5,1,4,6,7]:
    print(f"{names[k]:30s} {np.mean(t[:,k]-t[:,0]):9.0f}")
