"""Von Neumann amplification of the fully discrete scheme (R25) for cfg 2."""
import numpy as np, sys
sys.path.insert(0,'.')
import oracle
from fractions import Fraction
def gam(K,which): return oracle.gamma_row(K,which)
def Hspline(k, s, dx):
    # cubic B-spline interpolation transfer: value at x+s of interpolant of e^{ikx}, divided by e^{ikx}
    u = s/dx; q = np.floor(u); t = u-q
    B = np.array([(1-t)**3/6, (3*t**3-6*t**2+4)/6, (-3*t**3+3*t**2+3*t+1)/6, t**3/6])
    phase = np.exp(1j*k*dx*(q + np.arange(-1,3)))
    num = (B*phase).sum()
    den = (np.exp(-1j*k*dx)+4+np.exp(1j*k*dx))/6
    return num/den
def amp(K, dt, dx, L, r, th, kk):
    a,w = oracle.gauss_hermite(L); w = w/np.sqrt(np.pi)
    gy, gz = gam(K,'y'), gam(K,'z')
    rho = []; sig=[]
    for j in range(1,K+1):
        s = np.sqrt(2*j*dt)*a
        H = np.array([Hspline(kk, si, dx) for si in s])
        rho.append((w*H).sum()); sig.append((w*s*H).sum())
    # unknown vector V^n = (y^n, z^n); recurrence M0 V^n = sum_j Mj V^{n+j}
    M0 = np.array([[1 + K*dt*gy[0]*r, K*dt*gy[0]*th],[0, gz[0]]], dtype=complex)
    Ms = []
    for j in range(1,K+1):
        Mj = np.zeros((2,2),dtype=complex)
        # y eq
        if j==K: Mj[0,0] += rho[j-1]
        Mj[0,0] += -K*dt*gy[j]*r*rho[j-1]; Mj[0,1] += -K*dt*gy[j]*th*rho[j-1]
        # z eq
        if j==1: Mj[1,1] += rho[0]
        Mj[1,0] += gz[j]*(-r*sig[j-1]); Mj[1,1] += gz[j]*(-th*sig[j-1] - rho[j-1])
        Ms.append(np.linalg.solve(M0, Mj))
    # companion
    n=2*K; C = np.zeros((n,n),dtype=complex)
    for j in range(K): C[0:2, 2*j:2*j+2] = Ms[j]
    for j in range(1,K): C[2*j:2*j+2, 2*(j-1):2*(j-1)+2] = np.eye(2)
    return max(abs(np.linalg.eigvals(C)))
T=0.33; N=256; dt=T/N; r=0.03; th=(0.05-0.03+0.04)/0.2
for P in [8193, 16385, 24827, 32769, 65536]:
    dx = 32/(P-1)
    ks = np.linspace(0, np.pi/dx, 400)
    for K in [1,3,4,6]:
        g = max(amp(K,dt,dx,16,r,th,k) for k in ks)
        print(P, K, round(g,4))
print('--- L=32')
for P in [24827, 65536]:
    dx = 32/(P-1)
    ks = np.linspace(0, np.pi/dx, 400)
    for K in [4,6]:
        gs = [amp(K,dt,dx,32,r,th,k) for k in ks]
        print(P, K, round(max(gs),4), ks[int(np.argmax(gs))]*dx/np.pi)
print('--- where unstable L=16 P=65536 K=6')
dx=32/65535; ks=np.linspace(0,np.pi/dx,400); gs=[amp(6,dt,dx,16,r,th,k) for k in ks]
i=int(np.argmax(gs)); print(ks[i], ks[i]*dx/np.pi, 'unstable band', ks[np.array(gs)>1.0001].min(), ks[np.array(gs)>1.0001].max())
print('--- th=0 (f=-ry only)')
for K in [6]:
    print(max(amp(K,dt,dx,16,r,0.0,k) for k in ks))
