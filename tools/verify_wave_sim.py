"""Wave model of the C3 verification's host chains ("End game of the
dynamic split"): T threads, serial chain units of U ms (a row-1 continuation; a whole
chain = 2U), chunk c's GPU row-0 state ready at 1.51 (c + 1) + 0.6 ms. Prints the
all-host makespan per thread count and the best (wait threshold, whole-chain deadline)
policy. Usage: python tools/verify_wave_sim.py T [U]"""
import heapq
import sys
U=float(sys.argv[2]) if len(sys.argv)>2 else 17.0; Wt=2*U; link=1.51; n=64; T=int(sys.argv[1]); rows0=97.0
def st(c): return link*(c+1)+0.6
def sim(Wn, whole_rule_deadline=rows0, idle_whole=True):
    lo,hi=0,n-1; free=[0.0]*T; ends=[]
    # initial
    order=[]
    for i in range(T):
        if i<Wn and lo<=hi: ends.append(Wt); free[i]=Wt; hi-=1
        else: free[i]=0.0
    while lo<=hi:
        i=min(range(T),key=lambda j:free[j]); t=free[i]
        if st(lo)<=t: s=t; free[i]=s+U; ends.append(free[i]); lo+=1
        elif idle_whole and t+Wt<=whole_rule_deadline: free[i]=t+Wt; ends.append(free[i]); hi-=1
        else:
            s=st(lo); free[i]=s+U; ends.append(free[i]); lo+=1
    return max(ends)
for Wn in range(0,15):
    print(Wn, round(sim(Wn),1), round(sim(Wn,idle_whole=False),1))
def sim2(theta, dl):
    lo,hi=0,n-1; free=[0.0]*T; ends=[]
    while lo<=hi:
        i=min(range(T),key=lambda j:free[j]); t=free[i]
        if st(lo)<=t+theta or t+Wt>dl: s=max(t,st(lo)); free[i]=s+U; lo+=1
        else: free[i]=t+Wt; hi-=1
        ends.append(free[i])
    return max(ends)
best=min((sim2(th,dl),th,dl) for th in [x*0.25 for x in range(0,60)] for dl in range(80,115))
print(best)
for th in [0,1,2,3,4,6,8]: print(th,[round(sim2(th,dl),1) for dl in (90,95,97,100,103)])
