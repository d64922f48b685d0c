import numpy as np, time, threading
a = np.ones(1<<27); b = np.empty_like(a)  # 1 GiB each
b[:] = a
t=time.time(); 
for _ in range(3): np.copyto(b, a)
el=(time.time()-t)/3; print("1-thread memcpy %.1f GB/s (copied bytes)" % (a.nbytes/el/1e9))
def part(i, T):
    n=a.size//T; np.copyto(b[i*n:(i+1)*n], a[i*n:(i+1)*n])
for T in (2,4,8,16):
    t=time.time()
    for _ in range(3):
        th=[threading.Thread(target=part, args=(i,T)) for i in range(T)]
        [x.start() for x in th]; [x.join() for x in th]
    el=(time.time()-t)/3; print("%d-thread memcpy %.1f GB/s" % (T, a.nbytes/el/1e9))
