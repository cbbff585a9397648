"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, word for word (bit-exact on every RNS word),
plus decryption against the float64 plaintext product (north-star tolerance 1e-4 at scale 2^40)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

DELTA = 2.0 ** 40


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def setup_c1(torch_cuda):
    from paper_2509_09424_b200 import Context
    o = oracle.Oracle(12, 3, 1, 3)
    skc, sk, pk = o.keygen(synth.SEED_BASE + 1)
    ctx = Context(12, 3, 1, 3)
    ctx.load_keys(sk_ntt=sk)
    return o, sk, pk, ctx


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def test_moduli_and_roots_match_oracle(setup_c1, torch_cuda):
    o, sk, pk, ctx = setup_c1
    assert ctx.moduli == o.moduli and ctx.psi == o.psi
    from paper_2509_09424_b200 import Context
    big = Context(16, 12, 4, 3)
    ob = oracle.Oracle(16, 12, 4, 3)
    assert big.moduli == ob.moduli and big.psi == ob.psi


@pytest.mark.parametrize("log_n,L,alpha", [(12, 3, 1), (16, 12, 4), (13, 2, 1), (8, 2, 1)])
def test_ntt_bit_exact(torch_cuda, log_n, L, alpha):
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    ctx = Context(log_n, L, alpha, max(1, -(-L // alpha)))
    o = oracle.Oracle(log_n, L, alpha, max(1, -(-L // alpha)))
    T = L + alpha
    rs = np.random.default_rng(log_n)
    rows = np.stack([rs.integers(0, o.moduli[i % T], o.n, dtype=np.uint64) for i in range(2 * T)])
    rows[0, :3] = 0
    rows[1, :3] = np.uint64(o.moduli[1] - 1)
    t = dev(torch, rows)
    ctx.ntt(t, list(range(T)))
    got = host(t)
    want = np.stack([o.ntt(i % T, rows[i]) for i in range(2 * T)])
    assert (got == want).all()
    ctx.ntt(t, list(range(T)), inverse=True)
    assert (host(t) == rows).all()


def test_ntt_n16_extreme_inputs(torch_cuda):
    """N'=2^16 (the FP64 passes, ntt_fp.cuh): structured extreme rows on every limb (narrow 40-bit and wide 50-bit),
    forward and inverse separately, against the oracle's definition."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    ctx = Context(16, 12, 4, 3)
    o = oracle.Oracle(16, 12, 4, 3)
    T = 16
    rows, limbs = [], []
    for li in range(T):
        q = o.moduli[li]
        pats = [np.full(o.n, q - 1, dtype=np.uint64), np.full(o.n, (q + 1) // 2, dtype=np.uint64),
                np.tile(np.array([0, q - 1], dtype=np.uint64), o.n // 2), np.zeros(o.n, dtype=np.uint64)]
        pats[3][0] = q - 1
        for p in pats:
            rows.append(p)
            limbs.append(li)
    rows = np.stack(rows)
    t = dev(torch, rows)
    ctx.ntt(t, limbs)
    assert (host(t) == np.stack([o.ntt(limbs[i], rows[i]) for i in range(len(rows))])).all()
    t = dev(torch, rows)
    ctx.ntt(t, limbs, inverse=True)
    assert (host(t) == np.stack([o.intt(limbs[i], rows[i]) for i in range(len(rows))])).all()


def test_ntt_n16_many_rows(torch_cuda):
    """N'=2^16, 203 rows over every limb of Q u P in a permuted period (the FP64 passes with the TMA block pass):
    forward and inverse against the oracle, every word."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    ctx = Context(16, 12, 4, 3)
    o = oracle.Oracle(16, 12, 4, 3)
    T = 16
    rs = np.random.default_rng(203)
    period = [(7 * i) % T for i in range(T)]                 # row i holds limb period[i % 16]
    limbs = [period[i % T] for i in range(203)]
    rows = np.stack([rs.integers(0, o.moduli[li], o.n, dtype=np.uint64) for li in limbs])
    t = dev(torch, rows)
    ctx.ntt(t, period)
    want = np.stack([o.ntt(limbs[i], rows[i]) for i in range(len(rows))])
    assert (host(t) == want).all()
    ctx.ntt(t, period, inverse=True)
    assert (host(t) == rows).all()
    ctx.close()


def _enc_cols(o, pk, X, level, seed):
    d = X.shape[1]
    m_res = np.stack([o.encode(X[:, j], level, DELTA) for j in range(d)])
    return o.encrypt_batch(np.arange(d, dtype=np.uint64) + np.uint64(seed), pk, level, m_res)


@pytest.mark.parametrize("kernel", [1, 2, 3, 4])
def test_pcmm_a_encrypted_c1_bit_exact_and_decrypts(setup_c1, torch_cuda, kernel):
    """C1: 16x16 BitNet layer on real pk-encryptions; every word == oracle; decrypt == X.W within 1e-4."""
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    X = synth.gen_X(synth.SEED_BASE + 1, 16, 16)
    W = synth.gen_W(synth.SEED_BASE + 101, 16, 16)
    x = _enc_cols(o, pk, X, 3, 7000)
    want = o.pcmm_a(x, W)
    xd = dev(torch, x)
    yd = torch.empty((16, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, W, yd, level=3, kernel=kernel)
    torch.cuda.synchronize()
    got = host(yd)
    assert (got == want).all()
    ref = X @ W.astype(np.float64)
    for i in range(16):
        z = ctx.decrypt_debug(yd, i, 3)
        assert np.max(np.abs(z[:16] - ref[:, i])) < 1e-4
        zo = o.decrypt(sk, want[i], DELTA)
        assert np.max(np.abs(z - zo)) < 1e-9


def test_layout_b_after_host_pipeline_regrowth(setup_c1, torch_cuda):
    """ctx-owned buffers keep their lifetimes across entry points: Layout B (ctx Layout-B buffer), then the
    host-staged pipeline growing its staging area twice, new device allocations, then Layout B again -- still
    bit-exact (a stray free of the Layout-B buffer on staging regrowth was a use-after-free)."""
    from paper_2509_09424_b200 import Context
    o, sk, pk, _ = setup_c1
    torch = torch_cuda
    ctx = Context(12, 3, 1, 3)
    s, d, m = 16, 16, 16
    k, n_in, B, G, rots = oracle.layout_b_plan(o.n, s, d, m, 0)
    x = synth.gen_words(6300, o.q, n_in, 3, o.n)
    W = synth.gen_W(6301, d, m)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, B, G)
    keys = np.stack([o.rotkey(6400 + i, g, sk) for i, g in enumerate(gk)])
    want = o.pcmm_b(x, W, s, k, B, gk, keys)
    ctx.load_keys(sk_ntt=sk, galois=gk, rot_keys=keys)
    xd = dev(torch, x)
    yd = torch.empty((m, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, W, yd, level=3, layout=1, block_s=s)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()
    for dd in (40, 300):
        xa = synth.gen_words(6500 + dd, o.q, dd, 3, o.n)
        Wa = synth.gen_W(6600 + dd, dd, 24)
        ya = np.zeros((24, 2, 3, o.n), np.uint64)
        ctx.pcmm_ternary_host(xa, ctx.weights(Wa), ya, level=3)
        torch.cuda.synchronize()
        assert (ya == o.pcmm_a(xa, Wa, nthreads=4)).all()
    filler = torch.full((64 << 20,), 7, dtype=torch.int64, device="cuda")
    yd.zero_()
    ctx.pcmm_ternary(xd, W, yd, level=3, layout=1, block_s=s)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()
    assert bool((filler == 7).all())


@pytest.mark.parametrize("kernel", [1, 2, 3, 4])
@pytest.mark.parametrize("d,m,level", [(37, 70, 3), (1, 1, 1), (64, 64, 2), (130, 3, 3), (5, 129, 1), (900, 200, 1)])
def test_pcmm_a_ragged_shapes(setup_c1, torch_cuda, d, m, level, kernel):
    """Ragged d (pipeline tail) and m (partial 64-output tile), random words incl. 0 and q-1."""
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    x = synth.gen_words(d * 1000 + m, o.q, d, level, o.n)
    x[0, 0, 0, :7] = 0
    x[-1, 1, level - 1, :7] = np.uint64(o.q[level - 1] - 1)
    W = synth.gen_W(d + m, d, m)
    want = o.pcmm_a(x, W, nthreads=4)
    xd = dev(torch, x)
    yd = torch.empty((m, 2, level, o.n), dtype=torch.int64, device="cuda")
    w = ctx.weights(W)
    ctx.pcmm_ternary(xd, w, yd, level=level, kernel=kernel)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()


@pytest.mark.parametrize("L,alpha", [(12, 4), (48, 16)])
def test_pcmm_a_paper_default_ring_n14(torch_cuda, L, alpha):
    """The paper's default N'=2^14 at l = 12 and its stated L = 48 (64 moduli, the ctx maximum):
    Layout A on uniform words == oracle, every word (bench's Table III shapes run in this configuration)."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(14, L, alpha, 3)
    ctx = Context(14, L, alpha, 3)
    assert ctx.moduli == o.moduli
    d, m = 70, 40
    x = synth.gen_words(1400 + L, o.q, d, L, o.n)
    W = synth.gen_W(1401 + L, d, m)
    want = o.pcmm_a(x, W, nthreads=4)
    yd = torch.empty((m, 2, L, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(dev(torch, x), W, yd, level=L)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()


@pytest.mark.parametrize("kernel", [1, 2, 3, 4])
def test_pcmm_host_staged_pipeline(setup_c1, torch_cuda, kernel):
    """ensi_pcmm_ternary_host (pinned host in/out, slice-pipelined) == oracle, every word."""
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    d, m = 40, 70
    x = synth.gen_words(4242, o.q, d, 3, o.n)
    W = synth.gen_W(4243, d, m)
    want = o.pcmm_a(x, W, nthreads=4)
    xh = torch.from_numpy(x.view(np.int64)).pin_memory()
    yh = torch.zeros((m, 2, 3, o.n), dtype=torch.int64).pin_memory()
    w = ctx.weights(W)
    for _ in range(2):
        ctx.pcmm_ternary_host(xh.numpy(), w, yh.numpy(), level=3, kernel=kernel)
        torch.cuda.synchronize()
        assert (yh.numpy().view(np.uint64) == want).all()
        yh.zero_()


@pytest.mark.parametrize("kernel", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["zero", "identity", "neg_identity", "permutation", "plus", "minus", "toy"])
def test_pcmm_a_edge_weights(setup_c1, torch_cuda, kind, kernel):
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    d = m = 4 if kind == "toy" else 96
    if kind == "toy":
        m = 2
    W = synth.edge_W(kind, d, m, seed=5)
    x = synth.gen_words(77, o.q, d, 3, o.n)
    x[:, :, :, :11] = np.uint64(0)
    for r in range(3):
        x[:, :, r, 11:20] = np.uint64(o.q[r] - 1)
    want = o.pcmm_a(x, W, nthreads=4)
    xd = dev(torch, x)
    yd = torch.empty((m, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, W, yd, level=3, kernel=kernel)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()


@pytest.mark.parametrize("kernel", [1, 2, 3, 4])
def test_pcmm_a_long_sum_lazy_reduction(setup_c1, torch_cuda, kernel):
    """d = 8300 > 8184 (intermediate reduction) with every word q-1 and W all +1 / -1 / mixed."""
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    d, m, level = 8300, 3, 1
    x = np.full((d, 2, level, o.n), np.uint64(o.q[0] - 1), dtype=np.uint64)
    W = np.ones((d, m), np.int8)
    W[:, 1] = -1
    W[::3, 2] = -1
    xd = dev(torch, x)
    yd = torch.empty((m, 2, level, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, W, yd, level=level, kernel=kernel)
    torch.cuda.synchronize()
    got = host(yd)
    q = o.q[0]
    s2 = int(np.sum(W[:, 2].astype(np.int64)))
    for i, coef in enumerate([d, -d, s2]):
        assert (got[i] == np.uint64((coef * (q - 1)) % q)).all()


@pytest.mark.parametrize("bits", [(60, 59), (51, 50)])
@pytest.mark.parametrize("kernel", [1, 2, 3, 0])
def test_pcmm_a_wide_moduli_long_sum(torch_cuda, kernel, bits):
    """Moduli just under 2^60 (the ctx maximum) with d = 8300 terms of q - 1: the CUDA-core path must reduce its
    int64 accumulators every 7 rows there (accum_rows_between_reductions), the tcgen05 path takes the 128-bit
    combine -- closed-form expected words (sum_j W_ji) (q - 1) mod q, and == the oracle on one column.  Moduli just
    under 2^51 / 2^50 take the CUDA-core FP64-pipe loop at its shortest reduction interval (2 / 6 rows)."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    m2n = 1 << 13
    q = [_primes_1mod(m2n, 1 << bits[0], 1)[0], _primes_1mod(m2n, 1 << bits[1], 1)[0]]
    p = [_primes_1mod(m2n, 1 << 60, 1, skip=1)[0]]
    ctx = Context(12, 2, 1, 2, q=q, p=p)
    d, m, level = 8300, 3, 2
    x = np.empty((d, 2, level, ctx.n), np.uint64)
    for r in range(level):
        x[:, :, r, :] = np.uint64(q[r] - 1)
    W = np.ones((d, m), np.int8)
    W[:, 1] = -1
    W[::3, 2] = -1
    yd = torch.empty((m, 2, level, ctx.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(dev(torch, x), W, yd, level=level, kernel=kernel)
    torch.cuda.synchronize()
    got = host(yd)
    for i in range(m):
        coef = int(np.sum(W[:, i].astype(np.int64)))
        for r in range(level):
            assert (got[i, :, r] == np.uint64((coef * (q[r] - 1)) % q[r])).all(), (i, r)
    o = oracle.Oracle(12, 2, 1, 2, q=q, p=p)
    xs = x[:40].copy()
    xs[::2, 0, 0, ::5] = np.uint64(0)
    Ws = synth.gen_W(14000, 40, 3)
    yd = torch.empty((3, 2, level, ctx.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(dev(torch, xs), Ws, yd, level=level, kernel=kernel)
    torch.cuda.synchronize()
    assert (host(yd) == o.pcmm_a(xs, Ws)).all()


def test_pcmm_a_small_modulus_takes_cuda_cores(torch_cuda):
    """A modulus below 2^32 is outside the tcgen05 epilogue's range: the default kernel falls back to the CUDA
    cores (still the oracle's words), and requesting tcgen05 explicitly is ENSI_EINVAL."""
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_EINVAL
    torch = torch_cuda
    m2n = 1 << 13
    q = [_primes_1mod(m2n, 1 << 31, 1)[0], _primes_1mod(m2n, 1 << 45, 1)[0]]
    p = [_primes_1mod(m2n, 1 << 50, 1)[0]]
    ctx = Context(12, 2, 1, 2, q=q, p=p)
    o = oracle.Oracle(12, 2, 1, 2, q=q, p=p)
    assert ctx.kernel_name(0, 2) == "cuda-core"
    x = synth.gen_words(14100, o.q, 300, 2, o.n)
    W = synth.gen_W(14101, 300, 70)
    yd = torch.empty((70, 2, 2, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(dev(torch, x), W, yd, level=2)
    torch.cuda.synchronize()
    assert (host(yd) == o.pcmm_a(x, W, nthreads=4)).all()
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary(dev(torch, x), W, yd, level=2, kernel=2)
    assert e.value.code == ENSI_EINVAL
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary(dev(torch, x), W, yd, level=2, kernel=5)
    assert e.value.code == ENSI_EINVAL


@pytest.mark.parametrize("L,alpha,dnum", [(18, 6, 3), (10, 2, 5)])
def test_rotation_generic_keyswitch_kernels(torch_cuda, L, alpha, dnum):
    """Parameter sets outside the specialised key-switching kernels' bounds: E = L + alpha = 24 > 16 extended limbs
    (generic FP64 ModUp / ModDown conversions, per-limb final combine) and beta = 5 > 4 digits (generic key inner
    product) -- hoisted rotations and a rescale, word for word against the oracle."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(12, L, alpha, dnum)
    ctx = Context(12, L, alpha, dnum)
    assert ctx.moduli == o.moduli
    skc, sk, pk = o.keygen(14200 + L)
    gs = [o.galois(3), o.galois(-77)]
    keys = np.stack([o.rotkey(14300 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    for level in (L, L - 1):
        ct = synth.gen_words(14400 + level, o.q, 1, level, o.n)[0]
        yd = torch.empty((2, 2, level, o.n), dtype=torch.int64, device="cuda")
        ctx.rotate_hoisted(dev(torch, ct[None]), gs, yd, level)
        torch.cuda.synchronize()
        assert (host(yd) == o.rotate_hoisted(ct, gs, keys)).all(), level
    x = synth.gen_words(14500, o.q, 2, L, o.n)
    yr = torch.empty((2, 2, L - 1, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(dev(torch, x), yr, L)
    torch.cuda.synchronize()
    assert (host(yr) == np.stack([o.rescale(x[c]) for c in range(2)])).all()


def test_pcmm_errors(setup_c1, torch_cuda):
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_ENOTTERNARY, ENSI_EDIM, ENSI_EINVAL
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    x = torch.zeros((4, 2, 3, o.n), dtype=torch.int64, device="cuda")
    y = torch.zeros((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    W = np.zeros((4, 2), np.int8)
    W[2, 1] = 2
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary(x, W, y, level=3)
    assert e.value.code == ENSI_ENOTTERNARY and "W[2][1]" in str(e.value)
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary(x, np.zeros((5, 2), np.int8), y, level=3)
    assert e.value.code == ENSI_EDIM
    with pytest.raises(EnsiError) as e:
        ctx.pcmm_ternary(x, np.zeros((4, 4), np.int8), x, level=3)
    assert e.value.code in (ENSI_EINVAL, ENSI_EDIM)


# ---------------------------------------------------------------- rotation / key switching

@pytest.fixture(scope="module")
def rot_setup(setup_c1):
    o, sk, pk, ctx = setup_c1
    rs = [1, 2, 5, 16, 33, 100, -1, 1000]
    gs = [o.galois(r) for r in rs]
    keys = np.stack([o.rotkey(9000 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    return o, sk, pk, ctx, gs, keys


@pytest.mark.parametrize("level", [3, 2, 1])
def test_rotate_hoisted_bit_exact(rot_setup, torch_cuda, level):
    o, sk, pk, ctx, gs, keys = rot_setup
    torch = torch_cuda
    z = np.random.default_rng(level).uniform(-1, 1, o.n // 2)
    ct = o.encrypt(31 + level, pk, level, o.encode(z, level, DELTA))
    want = o.rotate_hoisted(ct, gs, keys)
    xd = dev(torch, ct[None])
    yd = torch.empty((len(gs), 2, level, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(xd, gs, yd, level)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()
    got = ctx.decrypt_debug(yd, 0, level)
    assert np.max(np.abs(got - np.roll(z, -1))) < 1e-5


@pytest.mark.parametrize("n_ct,sel", [(3, [0, 3]), (40, [5]), (5, [1, 2, 3, 4, 5, 6, 7])])
def test_rotate_batch_bit_exact(rot_setup, torch_cuda, n_ct, sel):
    """ensi_rotate_batch: y[c * n_g + r] = Rot_{g_r}(x_c) == oracle single rotation, every word (several inputs
    share each key batch; n_g = 1 over 40 inputs is the non-hoisted batch case)."""
    o, sk, pk, ctx, gs, keys = rot_setup
    torch = torch_cuda
    x = synth.gen_words(7700 + n_ct, o.q, n_ct, 3, o.n)
    g_sel = [gs[i] for i in sel]
    yd = torch.empty((n_ct * len(sel), 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_batch(dev(torch, x), g_sel, yd, 3)
    torch.cuda.synchronize()
    got = host(yd)
    for c in range(n_ct):
        for r, i in enumerate(sel):
            if c < 3 or c == n_ct - 1:
                assert (got[c * len(sel) + r] == o.rotate(x[c], gs[i], keys[i])).all()


def test_rotate_hoisted_128_elements_two_streams(setup_c1, torch_cuda):
    """128 Galois elements in one ensi_rotate_hoisted call (the hoisted rotations/s bench shape): four key-switch
    batches of 32 that alternate between the two internal streams, each with its own (acc, z) scratch set -- every
    output word == the oracle's hoisted rotation (O10), and the last one decrypts to the cyclic shift."""
    from paper_2509_09424_b200 import Context
    o, sk, pk, _ = setup_c1
    torch = torch_cuda
    ctx = Context(12, 3, 1, 3)
    gs = [o.galois(r) for r in range(1, 129)]
    keys = np.stack([o.rotkey(12000 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    z = np.random.default_rng(128).uniform(-1, 1, o.n // 2)
    ct = o.encrypt(12500, pk, 3, o.encode(z, 3, DELTA))
    want = o.rotate_hoisted(ct, gs, keys)
    yd = torch.empty((128, 2, 3, o.n), dtype=torch.int64, device="cuda")
    for _ in range(2):                      # twice: the second call reuses both scratch sets
        yd.zero_()
        ctx.rotate_hoisted(dev(torch, ct[None]), gs, yd, 3)
        torch.cuda.synchronize()
        assert (host(yd) == want).all()
    got = ctx.decrypt_debug(yd, 127, 3)
    assert np.max(np.abs(got - np.roll(z, -128))) < 1e-5


def test_rotate_batch_multi_batch_two_streams(setup_c1, torch_cuda):
    """ensi_rotate_batch with 5 inputs x 40 Galois elements = 200 rotations > 96: key-switch batches of 19 elements
    (<= 96 rotations each) on the two internal streams -- all 200 outputs == the oracle."""
    from paper_2509_09424_b200 import Context
    o, sk, pk, _ = setup_c1
    torch = torch_cuda
    ctx = Context(12, 3, 1, 3)
    gs = [o.galois(r) for r in range(-20, 21) if r != 0]
    keys = np.stack([o.rotkey(13000 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    x = synth.gen_words(13500, o.q, 5, 3, o.n)
    yd = torch.empty((5 * len(gs), 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_batch(dev(torch, x), gs, yd, 3)
    torch.cuda.synchronize()
    got = host(yd).reshape(5, len(gs), 2, 3, o.n)
    for c in range(5):
        assert (got[c] == o.rotate_hoisted(x[c], gs, keys)).all()


def test_rotate_identity_element_copies(rot_setup, torch_cuda):
    o, sk, pk, ctx, gs, keys = rot_setup
    torch = torch_cuda
    ct = synth.gen_words(3, o.q, 1, 3, o.n)
    xd = dev(torch, ct)
    yd = torch.empty((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(xd, [1, gs[0]], yd, 3)
    torch.cuda.synchronize()
    got = host(yd)
    assert (got[0] == ct[0]).all()
    assert (got[1] == o.rotate(ct[0], gs[0], keys[0])).all()


def test_rotate_missing_key(rot_setup, torch_cuda):
    from paper_2509_09424_b200.ensi import EnsiError, ENSI_ENOKEY
    o, sk, pk, ctx, gs, keys = rot_setup
    torch = torch_cuda
    xd = torch.zeros((1, 2, 3, o.n), dtype=torch.int64, device="cuda")
    yd = torch.zeros((1, 2, 3, o.n), dtype=torch.int64, device="cuda")
    with pytest.raises(EnsiError) as e:
        ctx.rotate_hoisted(xd, [o.galois(7)], yd, 3)
    assert e.value.code == ENSI_ENOKEY


# ---------------------------------------------------------------- Layout B

@pytest.mark.parametrize("lazy", [False, True])
@pytest.mark.parametrize("d,m,B,s", [(16, 16, 0, 16), (16, 16, 4, 16), (20, 6, 4, 16), (100, 130, 4, 64)])
def test_pcmm_layout_b_bit_exact(setup_c1, torch_cuda, d, m, B, s, lazy):
    """Layout B (O11) on real encryptions, every output word == the oracle; (100, 130, 4, 64): 7 giant steps over 130
    outputs = two key-stationary chunks (96 + 34) each split over the two internal streams, with the running sum
    added in place by the final combine.  lazy: R19 (moddown_lazy) against the oracle's lazy form -- G = 4 and 8
    giant steps accumulate over Q_l u P and take one ModDown per output (words differ from the eager form)."""
    from paper_2509_09424_b200 import Context
    o, sk, pk, _ = setup_c1
    torch = torch_cuda
    ctx = Context(12, 3, 1, 3)
    k, n_in, B, G, rots = oracle.layout_b_plan(o.n, s, d, m, B)
    X = synth.gen_X(61 + d, s, d)
    W = synth.gen_W(62 + d, d, m)
    slots = o.n // 2
    cts = []
    for c in range(n_in):
        zz = np.zeros(slots)
        for b in range(k):
            col = c * k + b
            if col < d:
                zz[b * s:(b + 1) * s] = X[:, col]
        cts.append(o.encrypt(6100 + c, pk, 3, o.encode(zz, 3, DELTA)))
    x = np.stack(cts)
    gk = oracle.layout_b_galois(o.n, o.log_n, s, B, G)
    keys = np.stack([o.rotkey(6200 + i, g, sk) for i, g in enumerate(gk)])
    want = o.pcmm_b(x, W, s, k, B, gk, keys, lazy=lazy)
    ctx.load_keys(sk_ntt=sk, galois=gk, rot_keys=keys)
    xd = dev(torch, x)
    yd = torch.empty((m, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, W, yd, level=3, layout=1, block_s=s, baby=B, moddown_lazy=lazy)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()
    ref = X @ W.astype(np.float64)
    for i in range(m):
        zz = ctx.decrypt_debug(yd, i, 3)
        assert np.max(np.abs(zz[:s] - ref[:, i])) < 1e-4


# ---------------------------------------------------------------- rescale

@pytest.mark.parametrize("level", [3, 2])
def test_rescale_bit_exact(setup_c1, torch_cuda, level):
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    x = synth.gen_words(90 + level, o.q, 5, level, o.n)
    want = np.stack([o.rescale(x[c]) for c in range(5)])
    xd = dev(torch, x)
    yd = torch.empty((5, 2, level - 1, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(xd, yd, level)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()


def test_rescale_chunked_many(setup_c1, torch_cuda):
    """More ciphertexts than one rescale chunk (256): words on both sides of the chunk boundary == oracle."""
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    cnt = 300
    x = synth.gen_words(95, o.q, cnt, 3, o.n)
    yd = torch.empty((cnt, 2, 2, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(dev(torch, x), yd, 3)
    torch.cuda.synchronize()
    got = host(yd)
    for c in (0, 255, 256, cnt - 1):
        assert (got[c] == o.rescale(x[c])).all()


def test_pcmm_with_rescale_epilogue(setup_c1, torch_cuda):
    """Inputs at Delta^2 (un-rescaled products); PCMM then rescale == oracle PCMM then oracle rescale."""
    o, sk, pk, ctx = setup_c1
    torch = torch_cuda
    X = synth.gen_X(5, 16, 8)
    W = synth.gen_W(6, 8, 8)
    scale2 = DELTA * DELTA
    m_res = np.stack([o.encode(X[:, j], 3, scale2) for j in range(8)])
    x = o.encrypt_batch(np.arange(8, dtype=np.uint64) + np.uint64(40), pk, 3, m_res)
    want = np.stack([o.rescale(c) for c in o.pcmm_a(x, W)])
    xd = dev(torch, x)
    yd = torch.empty((8, 2, 2, o.n), dtype=torch.int64, device="cuda")
    ls = ctx.pcmm_ternary(xd, W, yd, level=3, rescale_out=True, log2_scale=80.0)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()
    ref = X @ W.astype(np.float64)
    z = ctx.decrypt_debug(yd, 3, 2, log2_scale=ls)
    assert np.max(np.abs(z[:16] - ref[:, 3])) < 1e-4


@pytest.mark.parametrize("L,alpha,dnum,level", [(4, 2, 2, 4), (4, 2, 2, 3), (5, 2, 3, 5)])
def test_rotate_hoisted_n16_reduced_limbs(torch_cuda, L, alpha, dnum, level):
    """N'=2^16 with few limbs: the FP64 key-switching kernels (constant-bank ModUp / ModDown conversions, the
    two-digit and partial-last-digit key inner products, the separate ModDown INTT / conversion / NTT / combine
    steps) bit-exact against the oracle, including the identity element."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(16, L, alpha, dnum)
    skc, sk, pk = o.keygen(4242)
    ctx = Context(16, L, alpha, dnum)
    gs = [o.galois(r) for r in (1, 128, 3000)]
    keys = np.stack([o.rotkey(900 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    ct = synth.gen_words(77 + level, o.q, 1, level, o.n)[0]
    want = o.rotate_hoisted(ct, [1] + gs, keys[[0] + list(range(3))])
    yd = torch.empty((4, 2, level, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(dev(torch, ct[None]), [1] + gs, yd, level)
    torch.cuda.synchronize()
    assert (host(yd) == want).all()


@pytest.mark.parametrize("kernel", [2, 4, 1])
@pytest.mark.parametrize("d,m", [(2048, 1200), (300, 2100), (3072, 96), (200, 1200), (768, 3100)])
def test_pcmm_a_block_shapes_streamed_a(torch_cuda, kernel, d, m):
    """C3-C5-like shapes at a small ring: d > 768 streams W^T per stage (no resident A), m > 1024 has more than
    four pair groups -- the (super-group, word tile) items dealt round-robin to every co-resident cluster, super-groups
    overhanging the padded W^T, resident W^T (d <= 768) reloaded where a cluster's items cross super-groups;
    sampled output columns against the oracle."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    o = oracle.Oracle(12, 2, 1, 2)
    ctx = Context(12, 2, 1, 2)
    x = synth.gen_words(d + 7 * m, o.q, d, 2, o.n)
    W = synth.gen_W(d * 3 + m, d, m)
    xd = dev(torch, x)
    yd = torch.empty((m, 2, 2, o.n), dtype=torch.int64, device="cuda")
    ctx.pcmm_ternary(xd, ctx.weights(W), yd, level=2, kernel=kernel)
    torch.cuda.synchronize()
    cols = sorted(set([0, 1, m // 3, m // 2 + 1, m - 2, m - 1]))
    want = o.pcmm_a(x, W, cols=cols, nthreads=8)
    assert (host(yd[cols]) == want).all()


def test_cuda_graph_capture_replay(setup_c1, rot_setup, torch_cuda):
    """The product path is capturable: Layout A (tensor-core accumulate) and hoisted rotations recorded into one
    CUDA graph on a side stream and replayed give the same words as the oracle (no host sync inside the calls)."""
    o, sk, pk, ctx, gs, keys = rot_setup
    torch = torch_cuda
    d, m = 40, 70
    x = synth.gen_words(8100, o.q, d, 3, o.n)
    W = synth.gen_W(8101, d, m)
    w = ctx.weights(W)
    xd = dev(torch, x)
    yd = torch.empty((m, 2, 3, o.n), dtype=torch.int64, device="cuda")
    rd = torch.empty((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    ctx.pcmm_ternary(xd, w, yd, level=3, stream=s)          # warm-up outside capture (lazy tables, scratch)
    ctx.rotate_hoisted(xd[:1], gs[:2], rd, 3, stream=s)
    torch.cuda.synchronize()
    yd.zero_()
    rd.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.pcmm_ternary(xd, w, yd, level=3, stream=torch.cuda.current_stream())
        ctx.rotate_hoisted(xd[:1], gs[:2], rd, 3, stream=torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    assert (host(yd) == o.pcmm_a(x, W, nthreads=4)).all()
    assert (host(rd) == o.rotate_hoisted(x[0], gs[:2], keys[:2])).all()


def _primes_1mod(mod2n, below, count, skip=0):
    import sympy
    out, v = [], (below - 1) // mod2n * mod2n + 1
    while len(out) < count + skip:
        if v < below and sympy.isprime(v):
            out.append(v)
        v -= mod2n
    return out[skip:]


def test_custom_moduli_all_size_classes_n16(torch_cuda):
    """User-chosen moduli across the FP64 size classes at N'=2^16 (ntt_fp.cuh: 'wide' >= 2^41 incl. the largest
    below 2^50, 'narrow' just under 2^41, and a 31-bit prime): NTT both directions on extreme rows, hoisted
    rotations (ModUp / KIP / ModDown) and rescale, all word for word against the oracle."""
    from paper_2509_09424_b200 import Context
    torch = torch_cuda
    m2n = 1 << 17
    q = [_primes_1mod(m2n, 1 << 50, 1)[0], _primes_1mod(m2n, (1 << 41) + (1 << 36), 1)[0],
         _primes_1mod(m2n, 1 << 41, 1)[0], _primes_1mod(m2n, 1 << 31, 1)[0]]
    p = [_primes_1mod(m2n, 1 << 50, 1, skip=1)[0], _primes_1mod(m2n, 1 << 45, 1)[0]]
    o = oracle.Oracle(16, 4, 2, 2, q=q, p=p)
    ctx = Context(16, 4, 2, 2, q=q, p=p)
    assert ctx.moduli == o.moduli
    T = 6
    rows, limbs = [], []
    for li in range(T):
        qq = o.moduli[li]
        for pat in (np.full(o.n, qq - 1, np.uint64), np.tile(np.array([0, qq - 1], np.uint64), o.n // 2),
                    synth.gen_words(300 + li, [qq], 1, 1, o.n)[0, 0, 0]):
            rows.append(pat)
            limbs.append(li)
    rows = np.stack(rows)
    t = dev(torch, rows)
    ctx.ntt(t, limbs)
    assert (host(t) == np.stack([o.ntt(limbs[i], rows[i]) for i in range(len(rows))])).all()
    t = dev(torch, rows)
    ctx.ntt(t, limbs, inverse=True)
    assert (host(t) == np.stack([o.intt(limbs[i], rows[i]) for i in range(len(rows))])).all()
    skc, sk, pk = o.keygen(4242)
    gs = [o.galois(3), o.galois(1000)]
    keys = np.stack([o.rotkey(4300 + i, g, sk) for i, g in enumerate(gs)])
    ctx.load_keys(sk_ntt=sk, galois=gs, rot_keys=keys)
    ct = synth.gen_words(4400, o.q, 1, 4, o.n)[0]
    yd = torch.empty((2, 2, 4, o.n), dtype=torch.int64, device="cuda")
    ctx.rotate_hoisted(dev(torch, ct[None]), gs, yd, 4)
    torch.cuda.synchronize()
    assert (host(yd) == o.rotate_hoisted(ct, gs, keys)).all()
    x = synth.gen_words(4500, o.q, 2, 4, o.n)
    yr = torch.empty((2, 2, 3, o.n), dtype=torch.int64, device="cuda")
    ctx.rescale(dev(torch, x), yr, 4)
    torch.cuda.synchronize()
    assert (host(yr) == np.stack([o.rescale(x[c]) for c in range(2)])).all()


# ---------------------------------------------------------------- compact wire format (host transfers)

@pytest.mark.parametrize("log_n,L,alpha", [(12, 3, 1), (16, 12, 4)])
def test_wire_pack_unpack_device(torch_cuda, log_n, L, alpha):
    """Device pack / unpack == the numpy host serialisation (low ceil(bits/8) bytes of each word), both ways."""
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import wire_pack_host
    torch = torch_cuda
    ctx = Context(log_n, L, alpha, 3)
    x = synth.gen_words(9100 + log_n, ctx.q, 3, L, ctx.n)
    widths = ctx.wire_widths(L)
    want = wire_pack_host(x, widths)
    assert want.shape[1] == ctx.wire_bytes(L)
    out = torch.empty(want.size, dtype=torch.uint8, device="cuda")
    ctx.wire_pack(dev(torch, x), out, L)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == want.reshape(-1)).all()
    back = torch.empty((3, 2, L, ctx.n), dtype=torch.int64, device="cuda")
    ctx.wire_unpack(torch.from_numpy(want.reshape(-1)).cuda(), back, L)
    torch.cuda.synchronize()
    assert (host(back) == x).all()


def test_pcmm_host_wire_bit_exact(setup_c1, torch_cuda):
    """End-to-end PCMM on wire-format host buffers == the oracle (C1, real encryptions), and == the uint64 host
    path at C2 parameters on a 96 x 40 layer."""
    from paper_2509_09424_b200 import Context
    from paper_2509_09424_b200.ensi import wire_pack_host, wire_unpack_host
    o, sk, pk, ctx = setup_c1
    d, m = 24, 19
    X = synth.gen_X(9200, 16, d)
    W = synth.gen_W(9201, d, m)
    m_res = np.stack([o.encode(X[:, j], 3, DELTA) for j in range(d)])
    x = o.encrypt_batch(np.arange(d, dtype=np.uint64) + np.uint64(9300), pk, 3, m_res)
    widths = ctx.wire_widths(3)
    xw = wire_pack_host(x, widths)
    yw = np.zeros((m, ctx.wire_bytes(3)), np.uint8)
    w = ctx.weights(W)
    ctx.pcmm_ternary_host_wire(xw, w, yw, level=3)
    torch_cuda.cuda.synchronize()
    assert (wire_unpack_host(yw, widths, 3, o.n) == o.pcmm_a(x, W)).all()
    c2 = Context(16, 12, 4, 3)
    d, m = 96, 40
    x2 = synth.gen_words(9400, c2.q, d, 12, c2.n)
    W2 = synth.gen_W(9401, d, m)
    w2 = c2.weights(W2)
    y64 = np.zeros((m, 2, 12, c2.n), np.uint64)
    c2.pcmm_ternary_host(x2, w2, y64, level=12)
    w12 = c2.wire_widths(12)
    yw2 = np.zeros((m, c2.wire_bytes(12)), np.uint8)
    c2.pcmm_ternary_host_wire(wire_pack_host(x2, w12), w2, yw2, level=12)
    torch_cuda.cuda.synchronize()
    assert (wire_unpack_host(yw2, w12, 12, c2.n) == y64).all()
