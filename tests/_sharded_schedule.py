"""Test-side re-statement of libstr's mode-1-sharded two-pass STR step, run
with torch.distributed (gloo) on CPU.  Each rank holds rows [r*I_1/p, (r+1)*I_1/p) of mode 1 of
X_new, its own rows of G_1 / P_1, and replicas of everything else; the three data-path
exchanges are sum-allreduces at the same sites as the library:
  C1   partial M_N (t_new x R_N R_1)           after pass 1
  C2   partial Z_1 (from the local rows of G_1) after mode 1, and partial M_j for left modes j>1
  C2'  partial Y_R                              after pass 2
Matrices use the conventions of the library: slices G_n(i) are R_n x R_{n+1}; tables/Y entries
are row-major matrices; G_n(2) columns are r_n + R_n r_{n+1}.
"""
import numpy as np
import torch
import torch.distributed as dist


def _ar(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def slices(G):                                # paper core (R_n, I, R_{n+1}) -> (I, R_n, R_{n+1})
    return np.ascontiguousarray(G.transpose(1, 0, 2))


def chain_table(sl_list):
    """Products over the multi-index of the factors (first factor's index fastest)."""
    T = sl_list[0]
    for S in sl_list[1:]:
        T = np.einsum("xab,ybc->yxac", T, S).reshape(-1, T.shape[1], S.shape[2])
    return T


def zm(sl):                                   # Z as chain matrix [(a,c)][(b,d)] = sum_i G(b,a) G(d,c)
    I, Ra, Rb = sl.shape
    Z = np.einsum("iba,idc->acbd", sl, sl)     # (Rb, Rb, Ra, Ra) indexed [a, c, b, d]
    return Z.transpose(1, 0, 3, 2).reshape(Rb * Rb, Ra * Ra)   # row a + Rb c, col b + Ra d


def h2(Hm, Rn, Rn1):                          # H_<2>[i1 + Rn i2][r1 + Rn r2] = Hm[i1 + Rn r1][i2 + Rn1 r2]
    Q = np.empty((Rn * Rn1, Rn * Rn1))
    for i1 in range(Rn):
        for i2 in range(Rn1):
            for r1 in range(Rn):
                for r2 in range(Rn1):
                    Q[i1 + Rn * i2, r1 + Rn * r2] = Hm[i1 + Rn * r1, i2 + Rn1 * r2]
    return 0.5 * (Q + Q.T)


def to_g2(M):                                 # entries [b][a] (R_{n+1} x R_n) -> G(2) rows (a + R_n b)
    return M.reshape(M.shape[0], -1)


class ShardedSTR:
    """State of one rank.  cores: global paper-layout cores (the init), X_init: this rank's shard."""

    def __init__(self, cores, X_init_local, k, world, rank):
        self.N = len(cores)
        self.k, self.p, self.r = k, world, rank
        I1 = cores[0].shape[1]
        self.w = I1 // world
        self.sl = [slices(G) for G in cores]          # global slices (replicated), G_1 local rows below
        self.sl[0] = self.sl[0][rank * self.w:(rank + 1) * self.w]
        self.R = [G.shape[0] for G in cores]
        self._init(X_init_local)

    def Rn(self, n):
        return self.R[(n - 1) % self.N]

    def _Z(self, n):                                   # Z_n (Z_1 reduced over the shards)
        Z = zm(self.sl[n - 1])
        return _ar(Z) if n == 1 else Z

    def _chainH(self, n, Zs, ZN):
        """H^{≠n} chain matrix Z_{n-1} ... Z_1 ZN Z_{N-1} ... Z_{n+1} (Alg. 4 l.15)."""
        order = list(range(n - 1, 0, -1)) + [self.N] + list(range(self.N - 1, n, -1))
        H = None
        for j in order:
            Z = ZN if j == self.N else Zs[j - 1]
            H = Z if H is None else H @ Z
        return H

    def _contract(self, X, tn, GN_rows, init):
        """Pass 1 (old cores) and, on updates, the temporal solve (Alg. 4 l.8-10)."""
        N, k = self.N, self.k
        dims = [s.shape[0] for s in self.sl[:-1]]      # local I_1
        L = int(np.prod(dims[:k]))
        Rr = int(np.prod(dims[k:]))
        X3 = X.reshape(tn, Rr, L)                      # [t][r][l]
        TR = chain_table(self.sl[k:N - 1])             # (Rr, R_{k+1}, R_N)
        YL = np.einsum("trl,rpq->ltpq", X3, TR)        # (L, t, R_{k+1}, R_N)
        if not init:
            CL = chain_table(self.sl[:k])              # (L, R_1, R_{k+1}), local rows of G_1
            MN = _ar(np.einsum("lbc,ltca->tba", CL, YL))                      # site C1
            Zs = [self._Z(n) for n in range(1, N)]
            Hq = h2(self._chainN(Zs), self.Rn(N), self.Rn(1))
            GN_new = np.linalg.solve(Hq, to_g2(MN).T).T                       # (t, R_N R_1)
            GN_rows = GN_new.reshape(tn, self.Rn(1), self.Rn(N)).transpose(0, 2, 1)
        self.GN_rows = GN_rows
        W = np.einsum("ltca,tab->lcb", YL, GN_rows)    # (L, R_{k+1}, R_1)
        return W, X3, dims

    def _chainN(self, Zs):
        H = None
        for j in range(self.N - 1, 0, -1):
            H = Zs[j - 1] if H is None else H @ Zs[j - 1]
        return H

    def _modes(self, X, tn, GN_rows, W, X3, dims, ZN, accumulate):
        """Left modes from W, pass 2, right modes (Alg. 4 l.12-18 in the two-pass grouping)."""
        N, k = self.N, self.k
        Wl = W                                                   # index l = i_1 + I_1 i_2 + ...
        for j in range(1, N):
            if j <= k:
                # M_j(i_j) = sum_{l \\ i_j} (G_{j+1}..G_k)(old) W(l) (G_1..G_{j-1})(new)
                Lt = chain_table(self.sl[j:k]) if j < k else None           # (prod, R_{j+1}, R_{k+1})
                Rt = chain_table(self.sl[:j - 1]) if j > 1 else None        # (prod, R_1, R_j)
                M = np.zeros((dims[j - 1], self.Rn(j + 1), self.Rn(j)))
                for lidx in np.ndindex(*dims[:k]):
                    lin = 0
                    st = 1
                    for d, ii in zip(dims[:k], lidx):
                        lin += ii * st
                        st *= d
                    Wm = Wl[lin]
                    left_lin = 0
                    st = 1
                    for d, ii in zip(dims[j:k], lidx[j:k]):
                        left_lin += ii * st
                        st *= d
                    right_lin = 0
                    st = 1
                    for d, ii in zip(dims[:j - 1], lidx[:j - 1]):
                        right_lin += ii * st
                        st *= d
                    A = Lt[left_lin] if Lt is not None else np.eye(self.Rn(k + 1))
                    B = Rt[right_lin] if Rt is not None else np.eye(self.Rn(1))
                    M[lidx[j - 1]] += A @ Wm @ B
                if j > 1:
                    M = _ar(M)                                                 # site C2
            else:
                if j == k + 1:
                    TL = np.einsum("tab,lbc->tlac", GN_rows, chain_table(self.sl[:k])) \
                        if k > 0 else None                                     # (t, L, R_N, R_{k+1})
                    YR = _ar(np.einsum("trl,tlac->rac", X3, TL))              # site C2'
                    self.YR = YR
                Rd = dims[k:]
                Lt = chain_table(self.sl[j:N - 1]) if j < N - 1 else None      # (prod, R_{j+1}, R_N)
                Rt = chain_table(self.sl[k:j - 1]) if j > k + 1 else None      # (prod, R_{k+1}, R_j)
                M = np.zeros((dims[j - 1], self.Rn(j + 1), self.Rn(j)))
                for ridx in np.ndindex(*Rd):
                    lin = 0
                    st = 1
                    for d, ii in zip(Rd, ridx):
                        lin += ii * st
                        st *= d
                    pos = j - 1 - k
                    left_lin = 0
                    st = 1
                    for d, ii in zip(Rd[pos + 1:], ridx[pos + 1:]):
                        left_lin += ii * st
                        st *= d
                    right_lin = 0
                    st = 1
                    for d, ii in zip(Rd[:pos], ridx[:pos]):
                        right_lin += ii * st
                        st *= d
                    A = Lt[left_lin] if Lt is not None else np.eye(self.Rn(N))
                    B = Rt[right_lin] if Rt is not None else np.eye(self.Rn(k + 1))
                    M[ridx[pos]] += A @ self.YR[lin] @ B
            Mg2 = to_g2(M)
            self.P[j - 1] = Mg2 if not accumulate else self.P[j - 1] + Mg2
            Zs = [self._Z(n) for n in range(1, N)]
            H = self._chainH(j, Zs, ZN)
            Qn = h2(H, self.Rn(j), self.Rn(j + 1))
            self.Q[j - 1] = Qn if not accumulate else 0.5 * ((self.Q[j - 1] + Qn) + (self.Q[j - 1] + Qn).T)
            if accumulate:
                G2 = np.linalg.solve(self.Q[j - 1], self.P[j - 1].T).T
                self.sl[j - 1] = G2.reshape(-1, self.Rn(j + 1), self.Rn(j)).transpose(0, 2, 1)

    def _init(self, X):
        tn = X.shape[0]
        GN_rows = self.sl[-1]
        self.P = [None] * (self.N - 1)
        self.Q = [None] * (self.N - 1)
        W, X3, dims = self._contract(X, tn, GN_rows, init=True)
        self._modes(X, tn, GN_rows, W, X3, dims, zm(GN_rows), accumulate=False)

    def update(self, X):
        tn = X.shape[0]
        W, X3, dims = self._contract(X, tn, None, init=False)
        self.sl[-1] = np.concatenate([self.sl[-1], self.GN_rows], axis=0)
        self._modes(X, tn, self.GN_rows, W, X3, dims, zm(self.GN_rows), accumulate=True)

    def core(self, n):
        """Global paper-layout core n (G_1 gathered from the shards)."""
        s = self.sl[n - 1]
        if n == 1:
            parts = [torch.zeros_like(torch.from_numpy(s)) for _ in range(self.p)]
            dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(s)))
            s = np.concatenate([x.numpy() for x in parts], axis=0)
        return s.transpose(1, 0, 2)
