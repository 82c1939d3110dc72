"""CPU (numpy/scipy) implementations of the sharded path's local operations —
TEST INFRASTRUCTURE for the gloo world-size-2 tests of paper_2406_05020_b200.dist
(the product path uses the library kernels through GpuOps)."""
import numpy as np
import scipy.linalg as sl
import torch


class CpuOps:
    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64)

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=torch.float64)

    def kron(self, in_shape, out_shape, coefs, factors, x, y, nrhs, beta=0.0):
        X = x.numpy().reshape([nrhs] + list(in_shape))
        acc = 0.0
        for c, fs in zip(coefs, factors):
            Z = X
            for i, F in enumerate(fs):
                Z = np.moveaxis(np.tensordot(F.numpy(), Z, axes=([1], [i + 1])), 0, i + 1)
            acc = acc + c * Z
        Y = y.numpy().reshape([nrhs] + list(out_shape))
        Y[...] = acc + (beta * Y if beta else 0.0)

    def gemm(self, A, B, Cm, alpha=1.0, beta=0.0):
        Cm.numpy()[...] = alpha * (A.numpy() @ B.numpy()) + (beta * Cm.numpy() if beta else 0.0)

    def permute(self, src, shape, perm):
        return torch.from_numpy(np.ascontiguousarray(src.numpy().reshape(shape).transpose(perm)))

    def dots(self, X, v):
        return torch.from_numpy(X.numpy().reshape(X.shape[0], -1) @ v.numpy().reshape(-1))

    def axpy(self, y, X, coef, sign=1.0):
        y.numpy()[...] += sign * (coef.numpy() @ X.numpy().reshape(X.shape[0], -1)).reshape(y.shape)

    def vmul(self, x, d):
        x.numpy()[...] *= d.numpy()
        return x

    def transpose(self, A):
        return torch.from_numpy(np.ascontiguousarray(A.numpy().T))

    def fd_setup(self, ca, A0, A1, cb, B0, B1, noise):
        lam, V = sl.eigh(B0.numpy(), A0.numpy())
        mu, W = sl.eigh(A1.numpy(), B1.numpy())
        D = ca * mu[None, :] + cb * lam[:, None] + noise * np.outer((V * V).sum(0), (W * W).sum(0))
        return torch.from_numpy(V), torch.from_numpy(W), torch.from_numpy(1.0 / D)
