"""Test-only dense numpy model of the reference discretisation.

A third, independent implementation (besides the C++ oracle and the CUDA
product) of the assembled operators the reference's own tests build densely:
P1 mass/stiffness (src/assembly.cpp:31-103), Dirichlet reduction
(src/assembly.cpp:121-158), the flattened SG blocks (test_sg.cpp:294-309) and
the union-of-interiors Schur complement (test_dd.cpp:23-52, test_sg.cpp:115-141).
Small meshes only.
"""
import numpy as np


def mesh(nx, ny):
    npx = nx + 1
    i = np.tile(np.arange(nx + 1), ny + 1)
    j = np.repeat(np.arange(ny + 1), nx + 1)
    x, y = i / nx, j / ny
    elems = []
    for jj in range(ny):
        for ii in range(nx):
            a = jj * npx + ii
            b, c, d = a + 1, (jj + 1) * npx + ii + 1, (jj + 1) * npx + ii
            elems += [(a, b, c), (a, c, d)]
    bnd = (i == 0) | (i == nx) | (j == 0) | (j == ny)
    node_to_dof = -np.ones(len(x), int)
    free = np.where(~bnd)[0]
    node_to_dof[free] = np.arange(len(free))
    return x, y, np.array(elems), node_to_dof, free


def assemble(nx, ny, coeff=None, density=1.0):
    """Reduced dense (M, K) for a nodal coefficient (None -> mass only)."""
    x, y, el, n2d, free = mesh(nx, ny)
    n = len(free)
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    for e in el:
        x0, y0, x1, y1, x2, y2 = x[e[0]], y[e[0]], x[e[1]], y[e[1]], x[e[2]], y[e[2]]
        area = 0.5 * ((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0))
        b = np.array([y1 - y2, y2 - y0, y0 - y1])
        c = np.array([x2 - x1, x0 - x2, x1 - x0])
        g = (np.outer(b, b) + np.outer(c, c)) / (4 * area)
        m = density * area / 12 * (np.ones((3, 3)) + np.eye(3))
        cavg = 0.0 if coeff is None else (coeff[e[0]] + coeff[e[1]] + coeff[e[2]]) / 3
        for a in range(3):
            for bb in range(3):
                r, s = n2d[e[a]], n2d[e[bb]]
                if r < 0 or s < 0:
                    continue
                M[r, s] += m[a, bb]
                K[r, s] += cavg * g[a, bb]
    return M, K


def sg_blocks(nx, ny, coeff, tensor_dense):
    """(bigM, bigK) of the flattened SG system, term-major (test_sg.cpp:294-305)."""
    n_in, nt, _ = tensor_dense.shape
    M, _ = assemble(nx, ny)
    Ks = [assemble(nx, ny, coeff[i])[1] for i in range(n_in)]
    n = M.shape[0]
    bigM = np.kron(np.eye(nt), M)
    bigK = np.zeros((nt * n, nt * n))
    for i in range(n_in):
        bigK += np.kron(tensor_dense[i].T, Ks[i])  # block (k, j) += G_ijk K_i
    return bigM, bigK


def interface_split(nx, ny, px, py):
    """Reduced dof ids of the union of subdomain interiors and of the interface
    (structured partition, src/partition.cpp:48-133)."""
    x, y, el, n2d, free = mesh(nx, ny)
    owners = [set() for _ in range(len(x))]
    for e_id, e in enumerate(el):
        cx = (x[e[0]] + x[e[1]] + x[e[2]]) / 3
        cy = (y[e[0]] + y[e[1]] + y[e[2]]) / 3
        ci = min(nx - 1, int(cx * nx))
        cj = min(ny - 1, int(cy * ny))
        s = (cj * py // ny) * px + ci * px // nx
        for v in e:
            owners[v].add(s)
    iface = sorted(n2d[v] for v in range(len(x)) if len(owners[v]) >= 2 and n2d[v] >= 0)
    interior = sorted(n2d[v] for v in range(len(x)) if len(owners[v]) == 1 and n2d[v] >= 0)
    return np.array(interior, int), np.array(iface, int)


def newmark_dense(bigM, bigK, alpha0, alpha1, dt, u0, steps, zeta=0.25, gamma=0.5):
    """Plain dense Newmark loop of test_sg.cpp:306-333 (zero initial velocity)."""
    bigC = alpha0 * bigM + alpha1 * bigK
    mf, df = 1 / (zeta * dt * dt), gamma / (zeta * dt)
    Kt = mf * bigM + df * bigC + bigK
    u = u0.copy()
    v = np.zeros_like(u)
    a = np.linalg.solve(bigM, -bigC @ v - bigK @ u)
    out = [u.copy()]
    for _ in range(steps):
        um = (u + dt * v) / (zeta * dt * dt) + (1 - 2 * zeta) / (2 * zeta) * a
        uc = gamma * dt * um - v - (1 - gamma) * dt * a
        un = np.linalg.solve(Kt, bigM @ um + bigC @ uc)
        an = (un - u - dt * v) / (zeta * dt * dt) - (1 - 2 * zeta) / (2 * zeta) * a
        v = v + (1 - gamma) * dt * a + gamma * dt * an
        u, a = un, an
        out.append(u.copy())
    return out
