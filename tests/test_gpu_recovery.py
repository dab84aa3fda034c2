"""Recovery phase (§8f rank 4) on the GPU against the unmodified reference's
recover_inverse (oracle/_ref): bit-identical matrices, same errors.  Inputs
follow the reference's own tests (test_recovery.cpp): B_hat^{-1} from
dense_inverse of the augmented matrix, random dense matrices, zero plans,
singular updates."""
import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2409_03095_b200 import recovery
    return recovery, ref


def rand_dense(rng, n):
    return rng.uniform(-1, 1, (n, n))


def test_zero_plan_identity(env):  # test_recovery.cpp:33-38
    rec, ref = env
    m = rand_dense(np.random.default_rng(1), 5)
    out = rec.recover_inverse(m, np.zeros(5))
    assert bits_equal(out.ravel(), m.ravel())


@pytest.mark.parametrize("seed,n", [(0, 1), (1, 2), (2, 3), (3, 17), (4, 64), (5, 200), (6, 513)])
def test_random_plans_bit_exact(env, seed, n):
    rec, ref = env
    rng = np.random.default_rng(seed)
    m = rand_dense(rng, n) / n + np.eye(n)
    s = rng.uniform(-0.5, 0.5, n) * (rng.random(n) < 0.8)  # some zero entries (skipped updates)
    want = ref.recover_inverse(m, s)
    got = rec.recover_inverse(m, s)
    assert bits_equal(got.ravel(), want.ravel())


@pytest.mark.parametrize("kind", ["tridiag", "convdiff", "ddm"])
def test_augmented_split_roundtrip(env, kind):
    """B_hat^{-1} = dense_inverse(B + S) from the reference; recover with s."""
    rec, ref = env
    from paper_2409_03095_b200.recovery import csr_to_dense
    from paper_2409_03095_b200.mcspai import CsrMatrix
    r = {"tridiag": lambda: ref.gen_tridiagonal(40), "convdiff": lambda: ref.gen_convection_diffusion(9),
         "ddm": lambda: ref.gen_random_ddm(60, 0.2, 5)}[kind]()
    b = CsrMatrix(r.n, r.row_ptr, r.col_idx, r.values)
    d = csr_to_dense(b)
    bnorm = np.max(np.sum(np.abs(d), axis=1))
    s = np.where(np.diag(d) < 0, -1.0, 1.0) * 1.5 * bnorm
    bhat_inv = ref.dense_inverse(d + np.diag(s))
    want = ref.recover_inverse(bhat_inv, s)
    got = rec.recover_inverse(bhat_inv, s)
    assert bits_equal(got.ravel(), want.ravel())
    # and it is B^{-1} to rounding
    assert np.allclose(got @ d, np.eye(b.n), atol=1e-8)


def test_singular_update_and_args(env):
    rec, ref = env
    m = np.array([[1.0, 0.0], [0.0, 0.5]])
    s = np.array([0.0, 2.0])  # 1 - 2 * 0.5 == 0 at row 1 (test_recovery.cpp:91-96)
    with pytest.raises(rec.RecoveryError, match="singular update at row 1"):
        rec.recover_inverse(m, s)
    with pytest.raises(ref.RefError, match="row 1"):
        ref.recover_inverse(m, s)
    with pytest.raises(ValueError, match="recovery plan length mismatch"):
        rec.recover_inverse(m, np.zeros(3))
    with pytest.raises(ValueError, match="tol must be positive"):
        rec.recover_inverse(m, s, tol=0.0)


def test_device_inplace(env):
    import torch
    rec, ref = env
    rng = np.random.default_rng(9)
    n = 300
    m = rand_dense(rng, n) / n + np.eye(n)
    s = rng.uniform(-0.5, 0.5, n)
    t = torch.from_numpy(m.copy()).cuda()
    rec.recover_inverse_device(t, s)
    assert bits_equal(t.cpu().numpy().ravel(), ref.recover_inverse(m, s).ravel())
