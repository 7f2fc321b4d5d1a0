"""Readers of the reference-generated golden fixtures (tests/golden/) — test infrastructure."""


def unpack_case(z, key):
    W0 = z[key + "W0"]
    d, k = W0.shape
    ranks = [int(r) for r in z[key + "ranks"]]
    A_all, B_all = z[key + "A_all"], z[key + "B_all"]
    As, Bs, ao, bo = [], [], 0, 0
    for r in ranks:
        As.append(A_all[ao:ao + r * k].reshape(r, k))
        Bs.append(B_all[bo:bo + d * r].reshape(d, r))
        ao += r * k
        bo += d * r
    seqs, xo = [], 0
    X_all = z[key + "X_all"]
    for j, L in zip(z[key + "seq_job"], z[key + "seq_len"]):
        seqs.append((int(j), X_all[xo:xo + L * k].reshape(L, k)))
        xo += L * k
    return W0, ranks, As, Bs, seqs
