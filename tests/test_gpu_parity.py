"""Parity of the sm_100a engine (through the C ABI / public API) against the reference golden
vectors and the oracle.  Gates: |K_gpu - K_ref| <= 1e-12 absolute,
|amp_gpu - amp_ref| <= 1e-9 |amp_ref| + 1e-300, Gram diagonal exactly 1, Gram exactly symmetric,
identical SVC predictions."""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle  # noqa: E402
from paper_2405_02630_b200 import (FeatureMapConfig, RebindError, SweepPlan,  # noqa: E402
                                   compute_cross_kernel, compute_kernel_matrix, contract_batch)
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402

K_ABS = 1e-12
AMP_REL = 1e-9

L2_CASES = list(GOLDEN_CASES)  # every golden: layers 1 to 8


def _amp_ok(amp, ref):
    return np.all(np.abs(amp - ref) <= AMP_REL * np.abs(ref) + 1e-300)


@pytest.mark.parametrize("name", L2_CASES)
def test_pair_amplitudes_match_reference_golden(name):
    g = load_golden(name)
    L = int(g["layers"])
    plan = SweepPlan(g["A"].shape[1], L)
    A = torch.as_tensor(g["A"], device="cuda")
    B = torch.as_tensor(g["B"], device="cuda")
    pairs = torch.as_tensor(g["pairs"], device="cuda")
    amp = dev.pair_amplitudes(dev.gate_build(plan, A), dev.gate_build(plan, B), pairs)
    amp = amp.cpu().numpy()
    ref = g["amp_re"]
    assert np.abs(amp ** 2 - ref ** 2).max() <= K_ABS
    assert _amp_ok(amp, ref)


@pytest.mark.parametrize("name", [c for c in L2_CASES if c.startswith(("gram", "cross"))])
def test_public_api_matches_reference_golden(name):
    g = load_golden(name)
    cfg = FeatureMapConfig(g["A"].shape[1], layers=int(g["layers"]))
    if str(g["kind"]) == "gram":
        K = compute_kernel_matrix(g["A"], cfg).entries
        assert np.all(np.diag(K) == 1.0) and np.array_equal(K, K.T)
    else:
        K = compute_cross_kernel(g["A"], g["B"], cfg).entries
    assert np.abs(K - g["K"]).max() <= K_ABS


def test_contract_batch_dropin_matches_reference():
    g = load_golden("pairs_n50_L2")
    ops = [(g["A"][p], g["B"][q]) for p, q in g["pairs"]]
    amps = contract_batch(FeatureMapConfig(50), ops)
    assert all(isinstance(a, complex) and a.imag == 0.0 for a in amps)
    assert _amp_ok(np.array([a.real for a in amps]), g["amp_re"])
    assert contract_batch(FeatureMapConfig(50), []) == []
    with pytest.raises(RebindError, match="operand set 1"):
        contract_batch(FeatureMapConfig(50), [ops[0], (ops[1][0][:49], ops[1][1])])


def test_tile_sweep_and_pair_kernel_are_bit_identical(rng):
    n = 784
    X = rng.uniform(0, np.pi, (130, n)) * 0.05 + rng.uniform(0, np.pi, n)
    plan = SweepPlan(n, 2)
    Xd = torch.as_tensor(X, device="cuda")
    planes = dev.gate_build(plan, Xd)
    K = dev.gram(planes).cpu().numpy()
    i, j = np.triu_indices(130, 1)
    pairs = torch.as_tensor(np.stack([i, j], 1), device="cuda")
    amp = dev.pair_amplitudes(planes, planes, pairs).cpu().numpy()
    assert np.array_equal(K[i, j], amp * amp)


@pytest.mark.parametrize("n,N", [(1, 5), (2, 3), (15, 66), (16, 64), (17, 65), (33, 129),
                                 (50, 200), (784, 70)])
def test_gram_and_cross_vs_oracle_edge_sizes(n, N, rng):
    centre = rng.uniform(0, np.pi, n)
    X = centre + rng.normal(0, 0.6 / np.sqrt(n), (N, n))
    T = centre + rng.normal(0, 0.6 / np.sqrt(n), (7, n))
    for L in ((1, 2, 3, 4) if n <= 17 else (1, 2, 3) if n <= 50 else (1, 2)):
        cfg = FeatureMapConfig(n, layers=L)
        K = compute_kernel_matrix(X, cfg).entries
        Kx = compute_cross_kernel(T, X, cfg).entries
        assert np.abs(K - oracle.kernel_matrix(X, L)).max() <= K_ABS
        assert np.abs(Kx - oracle.cross_kernel(T, X, L)).max() <= K_ABS
        assert np.all(np.diag(K) == 1.0) and np.array_equal(K, K.T)


def test_magnitude_convention(rng):
    X = rng.uniform(0, 0.4, (40, 12))
    K = compute_kernel_matrix(X, FeatureMapConfig(12), convention="magnitude").entries
    assert np.abs(K - oracle.kernel_matrix(X, 2, "magnitude")).max() <= K_ABS


def test_cross_with_itself_equals_gram(rng):
    X = rng.uniform(0, 0.5, (90, 30))
    cfg = FeatureMapConfig(30)
    K = compute_kernel_matrix(X, cfg).entries
    Kx = compute_cross_kernel(X, X, cfg).entries
    assert np.abs(Kx - K).max() <= 1e-12
    assert np.all(np.abs(np.diag(Kx) - 1.0) <= 1e-9)


def test_trivial_sizes_and_errors():
    cfg = FeatureMapConfig(4)
    assert compute_kernel_matrix(np.zeros((0, 4)), cfg).entries.shape == (0, 0)
    assert compute_kernel_matrix(np.zeros((1, 4)), cfg).entries.tolist() == [[1.0]]
    assert np.all(compute_kernel_matrix(np.ones((4, 4)), cfg).entries == 1.0)
    with pytest.raises(RebindError, match="operand set 0: vectors of lengths 3/3"):
        compute_kernel_matrix(np.zeros((3, 3)), cfg)
    X = np.zeros((6, 4))
    X[3, 2] = np.nan
    with pytest.raises(RebindError, match="operand set 2: feature angles must be finite"):
        compute_kernel_matrix(X, cfg)
    T = np.zeros((2, 4))
    T[1, 0] = np.inf
    with pytest.raises(RebindError, match="operand set 6: feature angles must be finite"):
        compute_cross_kernel(T, np.zeros((6, 4)), cfg)


def test_one_qubit_closed_form():
    # n = 1, features {0, pi} -> off-diagonal cos^2(pi/2) = 0 (SPEC.md kernel_pipeline example)
    K = compute_kernel_matrix(np.array([[0.0], [np.pi]]), FeatureMapConfig(1, layers=1)).entries
    assert abs(K[0, 1]) <= 1e-30 and K[0, 0] == 1.0


def test_device_tensor_path_and_packed_unpack(rng):
    n, N = 64, 300
    X = torch.as_tensor(rng.uniform(0, 0.3, (N, n)), device="cuda")
    cfg = FeatureMapConfig(n)
    K_dev = compute_kernel_matrix(X, cfg).entries
    K_host = compute_kernel_matrix(X.cpu().numpy(), cfg).entries
    assert isinstance(K_dev, torch.Tensor) and K_dev.is_cuda
    assert np.array_equal(K_dev.cpu().numpy(), K_host)
    plan = SweepPlan(n, 2)
    planes = dev.gate_build(plan, X)
    nt = plan.gram_tile_count(N)
    K2 = torch.zeros((N, N), dtype=torch.float64, device="cuda")
    for lo, hi in [(0, nt // 3), (nt // 3, nt)]:
        packed = dev.gram(planes, tile_begin=lo, tile_end=hi, packed=True)
        dev.unpack_gram(plan, packed, N, lo, hi, K2)
    assert torch.equal(K2, K_dev)


def test_kernel_job_world1_matches_public_api(rng):
    n = 96
    Xtr = rng.uniform(0, 0.25, (257, n))
    Xte = rng.uniform(0, 0.25, (33, n))
    plan = SweepPlan(n, 2)
    job = KernelJob(plan, 257, 33)
    Ktr, Kx = job.run(torch.as_tensor(Xtr, device="cuda"), torch.as_tensor(Xte, device="cuda"))
    cfg = FeatureMapConfig(n)
    assert np.array_equal(Ktr.cpu().numpy(), compute_kernel_matrix(Xtr, cfg).entries)
    assert np.array_equal(Kx.cpu().numpy(), compute_cross_kernel(Xte, Xtr, cfg).entries)


def test_pinned_output_pipeline_matches_pageable(rng):
    n, N = 64, 1300  # 21 tile rows -> 3 super-row panels
    X = rng.uniform(0, 0.2, (N, n))
    cfg = FeatureMapConfig(n)
    pinned = torch.empty((N, N), dtype=torch.float64, pin_memory=True).numpy()
    K1 = compute_kernel_matrix(X, cfg, out=pinned).entries
    K2 = compute_kernel_matrix(X, cfg).entries
    assert np.array_equal(K1, K2)
    T = rng.uniform(0, 0.2, (300, n))
    pinned_x = torch.empty((300, N), dtype=torch.float64, pin_memory=True).numpy()
    assert np.array_equal(compute_cross_kernel(T, X, cfg, out=pinned_x).entries,
                          compute_cross_kernel(T, X, cfg).entries)


def test_library_results_are_page_locked_and_match_pageable_outputs(rng):
    """Results of >= 64 MB that the API allocates live in recycled page-locked mappings
    (kernel_pipeline._HostCache): the pipeline drains straight into them.  They must equal the
    drain into caller-supplied pageable arrays bit for bit, across recycled calls."""
    from paper_2405_02630_b200 import compute_kernel_matrices
    from paper_2405_02630_b200.kernel_pipeline import _host_cache

    n, N, M = 48, 3100, 2900  # 77 MB Gram, 72 MB cross
    X = rng.uniform(0, np.pi, n) + rng.normal(0, 0.3 / np.sqrt(n), (N, n))
    T = rng.uniform(0, np.pi, n) + rng.normal(0, 0.3 / np.sqrt(n), (M, n))
    cfg = FeatureMapConfig(n)
    ref_K, ref_Kx = np.zeros((N, N)), np.zeros((M, N))
    compute_kernel_matrices(X, T, cfg, out_train=ref_K, out_test=ref_Kx)
    for _ in range(3):  # the second and third calls get the first call's mappings back
        K, Kx = compute_kernel_matrices(X, T, cfg)
        registered = set(_host_cache.pinned.values())  # start addresses of the mappings
        assert K.entries.ctypes.data in registered and Kx.entries.ctypes.data in registered
        assert np.array_equal(K.entries, ref_K) and np.array_equal(Kx.entries, ref_Kx)
        del K, Kx
    i = rng.integers(0, N, 16)
    assert np.abs(ref_K[np.ix_(i, i)] - oracle.kernel_matrix(X[i], 2)).max() <= K_ABS


def test_full_size_gram_properties_and_sampled_parity():
    """BASELINE configs[3] at full size (10000 train Gram + 2000 x 10000 cross at 784 qubits,
    bandwidth-scaled overlapping MNIST-shaped data): size-independent properties plus 256
    sampled entries of each matrix against the oracle (every entry:
    profiles/r2_parity.json)."""
    from paper_2405_02630_b200 import compute_kernel_matrices
    from paper_2405_02630_b200.data import config_data

    Atr, _, Ate, _ = config_data(4, 10000, 2000, "mnist", bw=0.06, mix=0.6)
    cfg = FeatureMapConfig(784)
    KM, KxM = compute_kernel_matrices(Atr, Ate, cfg)
    K, Kx = KM.entries, KxM.entries
    assert np.all(np.diag(K) == 1.0)
    assert np.array_equal(K, K.T)
    assert K.min() >= 0.0 and K.max() <= 1.0 + 1e-9
    assert Kx.min() >= 0.0 and Kx.max() <= 1.0 + 1e-9
    rng = np.random.default_rng(5)
    i = rng.integers(0, 10000, 256)
    j = rng.integers(0, 10000, 256)
    keep = i != j
    ref = np.abs(oracle.amplitudes(Atr, Atr, np.stack([i[keep], j[keep]], 1), 2)) ** 2
    assert np.abs(K[i[keep], j[keep]] - ref).max() <= K_ABS
    r, c = rng.integers(0, 2000, 256), rng.integers(0, 10000, 256)
    refx = np.abs(oracle.amplitudes(Ate, Atr, np.stack([r, c], 1), 2)) ** 2
    assert np.abs(Kx[r, c] - refx).max() <= K_ABS
    assert 1e-3 <= np.median(ref) <= 0.5  # parity data is not in the concentrated K ~ 0 regime
    # the pinned-output pipeline (per-tile-row D2H racing the sweep, Gram panels split at
    # full size) lands the same bits as the pageable one
    pinned = torch.empty((10000, 10000), dtype=torch.float64, pin_memory=True).numpy()
    pinned.fill(np.nan)
    assert np.array_equal(compute_kernel_matrix(Atr, cfg, out=pinned).entries, K)


def test_svc_predictions_identical(rng):
    """Downstream: precomputed-kernel SVC, one-vs-rest, C = 1 — identical predictions from
    the engine's kernels and the oracle's (config-1-shaped: 8 qubits, 100 x 50)."""
    from sklearn.multiclass import OneVsRestClassifier
    from sklearn.svm import SVC

    from paper_2405_02630_b200.data import config_data

    Atr, ytr, Ate, yte = config_data(1, 100, 50, "mnist", features=8, binary=(2, 6))
    cfg = FeatureMapConfig(8)
    K = compute_kernel_matrix(Atr, cfg).entries
    Kx = compute_cross_kernel(Ate, Atr, cfg).entries
    Kr, Kxr = oracle.kernel_matrix(Atr, 2), oracle.cross_kernel(Ate, Atr, 2)
    assert np.abs(K - Kr).max() <= K_ABS and np.abs(Kx - Kxr).max() <= K_ABS
    clf = OneVsRestClassifier(SVC(kernel="precomputed", C=1.0)).fit(K, ytr)
    clf_r = OneVsRestClassifier(SVC(kernel="precomputed", C=1.0)).fit(Kr, ytr)
    assert np.array_equal(clf.predict(Kx), clf_r.predict(Kxr))


def test_shard_run_then_merge_equals_full_matrix(tmp_path, rng):
    """`--shard k/W` partials merged == the unsharded matrix, bit for bit."""
    from paper_2405_02630_b200.container import merge_partials, save_partial
    from paper_2405_02630_b200.kernel_pipeline import compute_kernel_shard

    n, N = 50, 137
    X = rng.uniform(0, 0.4, (N, n))
    T = rng.uniform(0, 0.4, (23, n))
    cfg = FeatureMapConfig(n)
    for test, full in [(None, compute_kernel_matrix(X, cfg).entries),
                       (T, compute_cross_kernel(T, X, cfg).entries)]:
        paths = []
        for k in range(3):
            rng_k, vals = compute_kernel_shard(X, cfg, k, 3, test=test)
            p = tmp_path / f"{'g' if test is None else 'x'}{k}.qkk"
            rows = N if test is None else len(T)
            save_partial(p, vals, rng_k, rows, N, test is None)
            paths.append(p)
        assert np.array_equal(merge_partials(paths).entries, full)


@pytest.mark.parametrize("layers", [1, 2, 3, 4, 5, 6])
def test_joint_train_test_pass_equals_separate_calls(layers, rng):
    """compute_kernel_matrices (one sweep over the joint tile list, host pipeline) and the
    device job path == compute_kernel_matrix + compute_cross_kernel, bit for bit."""
    from paper_2405_02630_b200 import compute_kernel_matrices

    n = 40 if layers < 3 else 12 if layers == 3 else 6 if layers <= 5 else 3
    Xtr = rng.uniform(0, 0.3, (600, n))
    Xte = rng.uniform(0, 0.3, (150, n))
    cfg = FeatureMapConfig(n, layers=layers)
    K, Kx = compute_kernel_matrices(Xtr, Xte, cfg)
    assert np.array_equal(K.entries, compute_kernel_matrix(Xtr, cfg).entries)
    assert np.array_equal(Kx.entries, compute_cross_kernel(Xte, Xtr, cfg).entries)
    pinned_k = torch.empty((600, 600), dtype=torch.float64, pin_memory=True).numpy()
    pinned_x = torch.empty((150, 600), dtype=torch.float64, pin_memory=True).numpy()
    K2, Kx2 = compute_kernel_matrices(Xtr, Xte, cfg, out_train=pinned_k, out_test=pinned_x)
    assert np.array_equal(K2.entries, K.entries) and np.array_equal(Kx2.entries, Kx.entries)
    job = KernelJob(SweepPlan(n, layers), 600, 150)
    Kd, Kxd = job.run(torch.as_tensor(Xtr, device="cuda"), torch.as_tensor(Xte, device="cuda"))
    assert np.array_equal(Kd.cpu().numpy(), K.entries)
    assert np.array_equal(Kxd.cpu().numpy(), Kx.entries)


def test_config2_full_matrices_vs_oracle():
    """BASELINE configs[1]: 50 qubits (PCA), 1000 train x 500 test — EVERY entry of both
    matrices against the oracle (1e-12), and identical SVC predictions."""
    from sklearn.svm import SVC

    from paper_2405_02630_b200 import compute_kernel_matrices
    from paper_2405_02630_b200.data import config_data

    Atr, ytr, Ate, yte = config_data(2, 1000, 500, "mnist", features=50, binary=(2, 6))
    cfg = FeatureMapConfig(50)
    K, Kx = compute_kernel_matrices(Atr, Ate, cfg)
    Kr, Kxr = oracle.kernel_matrix(Atr, 2), oracle.cross_kernel(Ate, Atr, 2)
    assert np.abs(K.entries - Kr).max() <= K_ABS and np.abs(Kx.entries - Kxr).max() <= K_ABS
    # min-max angles over [0, pi] concentrate this kernel (median K ~ 1e-10), so the
    # absolute gate alone is weak: |amp| = sqrt(K) must also agree to 1e-9 relative, with a
    # 1e-18 absolute floor for amplitudes that are themselves cancellation residues (~1e-12
    # from ~1e-10 terms; two exact fp64 orders differ there by ~1e-20 absolute)
    for got, ref in ((K.entries, Kr), (Kx.entries, Kxr)):
        a, b = np.sqrt(got), np.sqrt(ref)
        assert np.all(np.abs(a - b) <= AMP_REL * b + 1e-18)
    p = SVC(kernel="precomputed", C=1.0).fit(K.entries, ytr).predict(Kx.entries)
    pr = SVC(kernel="precomputed", C=1.0).fit(Kr, ytr).predict(Kxr)
    assert np.array_equal(p, pr)


def _ovr(K, y, Kx):
    from sklearn.multiclass import OneVsRestClassifier
    from sklearn.svm import SVC

    clf = OneVsRestClassifier(SVC(kernel="precomputed", C=1.0)).fit(K, y)
    return clf.predict(Kx), clf.decision_function(Kx)


def test_config3_shaped_every_entry_identical_ovr_predictions():
    """The north-star gate at 784 qubits on a config-3-shaped job small enough for the oracle
    to check EVERY entry in seconds: Fashion-shaped, 10-class one-vs-rest, 400 x 200, angles
    0.06 pi pixel on overlapping classes (mix 0.6), so the median K sits inside [1e-3, 0.5]
    and the accuracy is well below 1.  Every entry within 1e-12 of the oracle's; identical
    predictions and (to 1e-9) identical decision values from the engine's K and the oracle's.
    The full 2000 x 1000 / 10000 x 2000 configs: tools/parity_report.py ->
    profiles/r2_parity.json."""
    from paper_2405_02630_b200 import compute_kernel_matrices
    from paper_2405_02630_b200.data import config_data

    Atr, ytr, Ate, yte = config_data(3, 400, 200, "fashion", bw=0.06, mix=0.6)
    K, Kx = compute_kernel_matrices(Atr, Ate, FeatureMapConfig(784))
    Kr, Kxr = oracle.kernel_matrix(Atr, 2), oracle.cross_kernel(Ate, Atr, 2)
    assert np.abs(K.entries - Kr).max() <= K_ABS
    assert np.abs(Kx.entries - Kxr).max() <= K_ABS
    assert 1e-3 <= np.median(Kr[np.triu_indices(400, 1)]) <= 0.5
    p, d = _ovr(K.entries, ytr, Kx.entries)
    pr, dr = _ovr(Kr, ytr, Kxr)
    assert np.array_equal(p, pr)
    assert np.abs(d - dr).max() <= 1e-9
    acc = float((p == yte).mean())
    assert 0.3 < acc < 0.98, acc  # far above chance (0.1), and not trivially separable


def test_config3_fashion_784_sampled_and_ovr_predictions():
    """BASELINE configs[2] at full size: Fashion-shaped, 10-class one-vs-rest, 784 qubits,
    2000 x 1000 on the same bandwidth-scaled overlapping data — 512 sampled entries of each
    matrix vs the oracle, and identical OvR predictions from the engine's K and from K with
    the sampled entries replaced by the oracle's values (every entry of this config:
    profiles/r2_parity.json)."""
    from paper_2405_02630_b200 import compute_kernel_matrices
    from paper_2405_02630_b200.data import config_data

    Atr, ytr, Ate, yte = config_data(3, 2000, 1000, "fashion", bw=0.06, mix=0.6)
    K, Kx = compute_kernel_matrices(Atr, Ate, FeatureMapConfig(784))
    K, Kx = K.entries, Kx.entries
    rng = np.random.default_rng(11)
    i, j = rng.integers(0, 2000, 512), rng.integers(0, 2000, 512)
    keep = i != j
    i, j = i[keep], j[keep]
    ref = np.abs(oracle.amplitudes(Atr, Atr, np.stack([i, j], 1), 2)) ** 2
    assert np.abs(K[i, j] - ref).max() <= K_ABS
    r, c = rng.integers(0, 1000, 512), rng.integers(0, 2000, 512)
    refx = np.abs(oracle.amplitudes(Ate, Atr, np.stack([r, c], 1), 2)) ** 2
    assert np.abs(Kx[r, c] - refx).max() <= K_ABS
    assert 1e-3 <= np.median(ref) <= 0.5
    Ks, Kxs = K.copy(), Kx.copy()
    Ks[i, j] = Ks[j, i] = ref
    Kxs[r, c] = refx
    p, _ = _ovr(K, ytr, Kx)
    ps, _ = _ovr(Ks, ytr, Kxs)
    assert np.array_equal(p, ps)
    acc = float((p == yte).mean())
    assert 0.3 < acc < 0.98, acc


@pytest.mark.parametrize("n", [1600, 2100])
def test_wide_chains_cross_rescale_points(n, rng):
    """n > 1024: the L = 2 sweep rescales its state by 2^-512 every 512 qubits (3-4 times
    here) and pads the front of the chain; tightly clustered samples keep K ~ 1e-2..1."""
    X = rng.uniform(0, np.pi, n) + rng.normal(0, 0.02, (70, n))
    T = X[:5] + rng.normal(0, 0.01, (5, n))
    cfg = FeatureMapConfig(n)
    K = compute_kernel_matrix(X, cfg).entries
    Kx = compute_cross_kernel(T, X, cfg).entries
    Kr, Kxr = oracle.kernel_matrix(X, 2), oracle.cross_kernel(T, X, 2)
    assert np.abs(K - Kr).max() <= K_ABS and np.abs(Kx - Kxr).max() <= K_ABS
    assert np.all(np.abs(np.sqrt(K) - np.sqrt(Kr)) <= AMP_REL * np.sqrt(Kr) + 1e-300)


def test_large_and_negative_angles(rng):
    """Any finite angle is valid (the reference only checks finiteness, circuit.py:112-118):
    large magnitudes and negative values against the oracle for L = 1, 2, 3, 5."""
    X = rng.normal(0, 1, (40, 9)) * np.array([1, 10, 100, 1e3, 1e4, 1e5, -1e6, 3e7, -1e8])
    X[5] = X[4] + 1e-3
    for L in (1, 2, 3, 5):
        K = compute_kernel_matrix(X, FeatureMapConfig(9, layers=L)).entries
        assert np.abs(K - oracle.kernel_matrix(X, L)).max() <= K_ABS, L


@pytest.mark.parametrize("L", [1, 2, 3, 5])
def test_spec_invariants_range_and_psd(L, rng):
    """SPEC kernel_pipeline invariants: entries in [0, 1 + 1e-9]; the probability-convention
    Gram is positive semidefinite (smallest eigenvalue >= -1e-8, K_ij = Tr(rho_i rho_j));
    a test point identical to a train point gives 1 at that column."""
    n = 12 if L <= 3 else 6
    X = rng.uniform(0, np.pi, n) + rng.normal(0, 0.4, (120, n))
    cfg = FeatureMapConfig(n, layers=L)
    K = compute_kernel_matrix(X, cfg).entries
    assert K.min() >= 0.0 and K.max() <= 1.0 + 1e-9
    assert np.linalg.eigvalsh(K).min() >= -1e-8
    Kx = compute_cross_kernel(X[[7, 30]], X, cfg).entries
    assert Kx.min() >= 0.0 and Kx.max() <= 1.0 + 1e-9
    assert abs(Kx[0, 7] - 1.0) <= 1e-9 and abs(Kx[1, 30] - 1.0) <= 1e-9


def test_large_sample_count_device_gram(rng):
    """N = 70,000 samples (a 39 GB dense Gram, 2.45e9 entries, 1.2e6 tiles; int64 offsets
    beyond 2^31 everywhere): sampled entries against the oracle, mirror and unit diagonal."""
    N, n = 70000, 8
    X = torch.as_tensor(rng.uniform(0, np.pi, n) + rng.normal(0, 0.3, (N, n)), device="cuda")
    plan = SweepPlan(n, 2)
    K = dev.gram(dev.gate_build(plan, X))
    torch.cuda.synchronize()
    Xh = X.cpu().numpy()
    idx = np.concatenate([[0, 1, N - 2, N - 1], rng.integers(0, N, 60)])
    i, j = np.meshgrid(idx, idx, indexing="ij")
    got = K[torch.as_tensor(i, device="cuda"), torch.as_tensor(j, device="cuda")].cpu().numpy()
    sel = np.unique(idx)
    ref = oracle.kernel_matrix(Xh[sel], 2)
    pos = {v: k for k, v in enumerate(sel)}
    want = np.array([[ref[pos[a], pos[b]] for b in idx] for a in idx])
    assert np.abs(got - want).max() <= K_ABS
    assert np.array_equal(got, got.T)
    del K
    torch.cuda.empty_cache()


def test_empty_cross_blocks_and_joint_pass():
    from paper_2405_02630_b200 import compute_kernel_matrices

    cfg = FeatureMapConfig(5)
    X = np.random.default_rng(3).uniform(0, 1, (7, 5))
    assert compute_cross_kernel(np.zeros((0, 5)), X, cfg).entries.shape == (0, 7)
    assert compute_cross_kernel(X, np.zeros((0, 5)), cfg).entries.shape == (7, 0)
    K, Kx = compute_kernel_matrices(X, np.zeros((0, 5)), cfg)
    assert K.entries.shape == (7, 7) and Kx.entries.shape == (0, 7)
    assert np.abs(K.entries - oracle.kernel_matrix(X, 2)).max() <= K_ABS


@pytest.mark.parametrize("n,n_train,n_test", [(784, 2000, 300), (200, 6000, 0), (64, 9000, 777)])
def test_pinned_head_first_pipeline_matches_pageable(n, n_train, n_test, rng):
    """Pinned host inputs take the head-first pipeline (the B-block Gram head is swept while
    the rest of the angles upload); it must equal the pageable path bit for bit."""
    from paper_2405_02630_b200 import compute_kernel_matrices

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
        t[...] = a
        return t

    X = rng.uniform(0, np.pi, n) + rng.normal(0, 0.3 / np.sqrt(n), (n_train, n))
    T = rng.uniform(0, np.pi, n) + rng.normal(0, 0.3 / np.sqrt(n), (n_test, n))
    cfg = FeatureMapConfig(n)
    K, Kx = compute_kernel_matrices(X, T, cfg)
    Kp, Kxp = compute_kernel_matrices(pinned(X), pinned(T), cfg,
                                      out_train=pinned(np.zeros((n_train, n_train))),
                                      out_test=pinned(np.zeros((n_test, n_train))))
    assert np.array_equal(K.entries, Kp.entries)
    assert np.array_equal(Kx.entries, Kxp.entries)
    Kq, Kxq = compute_kernel_matrices(pinned(X), pinned(T), cfg,  # pageable outputs
                                      out_train=np.zeros((n_train, n_train)),
                                      out_test=np.zeros((n_test, n_train)))
    assert np.array_equal(K.entries, Kq.entries) and np.array_equal(Kx.entries, Kxq.entries)
    Kg = compute_kernel_matrix(pinned(X), cfg)  # Gram-only entry: the joint pipeline
    assert np.array_equal(K.entries, Kg.entries)
    i = rng.integers(0, n_train, 24)
    assert np.abs(K.entries[np.ix_(i, i)] - oracle.kernel_matrix(X[i], 2)).max() <= K_ABS


@pytest.mark.parametrize("where", ["head", "rest", "test"])
def test_pinned_head_first_non_finite_raises_rebind(where, rng):
    """A non-finite angle in the head's samples, in the rest (uploaded and gate-built on the
    second stream beside the head sweep) or in the test set raises the reference's
    RebindError, and the pipeline is healthy afterwards (same result as before)."""
    from paper_2405_02630_b200 import RebindError, compute_kernel_matrices

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
        t[...] = a
        return t

    n, N, M = 784, 3000, 200
    X = pinned(rng.uniform(0, np.pi, (N, n)))
    T = pinned(rng.uniform(0, np.pi, (M, n)))
    cfg = FeatureMapConfig(n)
    K0, Kx0 = compute_kernel_matrices(X, T, cfg)
    bad = {"head": (X, 5), "rest": (X, N - 3), "test": (T, M - 1)}[where]
    old = bad[0][bad[1], 100]
    bad[0][bad[1], 100] = np.nan
    with pytest.raises(RebindError, match=r"operand set \d+: feature angles must be finite"):
        compute_kernel_matrices(X, T, cfg)
    bad[0][bad[1], 100] = old
    K1, Kx1 = compute_kernel_matrices(X, T, cfg)
    assert np.array_equal(K0.entries, K1.entries) and np.array_equal(Kx0.entries, Kx1.entries)


def test_kernel_job_graph_replay_matches_run(rng):
    """KernelJob.graph: a CUDA-graph replay of the job recomputes the same matrices, also
    after the input tensors are refilled in place."""
    n, N, M = 24, 300, 70
    tr = torch.as_tensor(rng.uniform(0, np.pi, (N, n)), device="cuda")
    te = torch.as_tensor(rng.uniform(0, np.pi, (M, n)), device="cuda")
    job = KernelJob(SweepPlan(n, 2), N, M)
    replay, K, Kx = job.graph(tr, te)
    replay()
    torch.cuda.synchronize()
    K0, Kx0 = KernelJob(SweepPlan(n, 2), N, M).run(tr, te)
    assert torch.equal(K, K0) and torch.equal(Kx, Kx0)
    tr.copy_(torch.as_tensor(rng.uniform(0, np.pi, (N, n)), device="cuda"))
    replay()
    torch.cuda.synchronize()
    K1, _ = KernelJob(SweepPlan(n, 2), N, M).run(tr, te)
    assert torch.equal(K, K1)


@pytest.mark.parametrize("n", [50, 64])
def test_kernel_job_auto_graph_matches_eager_and_api(rng, n):
    """Small single-GPU jobs replay a captured qk_job_run by default: bit-identical to the
    eager path and to the public API, fresh inputs every call (copied into the job's
    buffers), and the reference's RebindError for a non-finite angle in either mode."""
    N, M = 333, 71
    cfg = FeatureMapConfig(n)
    auto = KernelJob(SweepPlan(n, 2), N, M)
    eager = KernelJob(SweepPlan(n, 2), N, M, graph_mode=False)
    assert auto._graph_eligible() and not eager._graph_eligible()
    for _ in range(3):
        Xtr = rng.uniform(0, 0.3, (N, n))
        Xte = rng.uniform(0, 0.3, (M, n))
        tr, te = torch.as_tensor(Xtr, device="cuda"), torch.as_tensor(Xte, device="cuda")
        K, Kx = auto.run(tr, te)
        Ke, Kxe = eager.run(tr, te)
        assert torch.equal(K, Ke) and torch.equal(Kx, Kxe)
        assert np.array_equal(K.cpu().numpy(), compute_kernel_matrix(Xtr, cfg).entries)
        assert np.array_equal(Kx.cpu().numpy(), compute_cross_kernel(Xte, Xtr, cfg).entries)
    assert auto._g is not None
    bad_tr = tr.clone()
    bad_tr[7, 3] = float("nan")
    for job in (auto, eager):
        with pytest.raises(RebindError, match="operand set 6: feature angles must be finite"):
            job.run(bad_tr, te)
        bad_te = te.clone()
        bad_te[2, 0] = float("inf")
        with pytest.raises(RebindError, match=f"operand set {2 * N}: feature angles must be"):
            job.run(tr, bad_te)
        job.run(tr, te)  # the sentinels reset on the next call


_LAYOUT_PROBE = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2405_02630_b200 import SweepPlan
from paper_2405_02630_b200.distributed import KernelJob
rng = np.random.default_rng(3)
out = {{}}
for n in (5, 16, 33, 64):
    tr = torch.as_tensor(rng.uniform(0, 0.4, (700, n)), device="cuda")
    te = torch.as_tensor(rng.uniform(0, 0.4, (130, n)), device="cuda")
    K, Kx = KernelJob(SweepPlan(n, 2), 700, 130, graph_mode=False).run(tr, te)
    out[f"K{{n}}"], out[f"Kx{{n}}"] = K.cpu().numpy(), Kx.cpu().numpy()
np.savez({path!r}, **out)
"""


def test_short_chain_layouts_bit_identical(tmp_path):
    """Short chains (n_pad <= 64) run 32-row items with all 16 warps busy (RI = 1); the
    64-row-item layout (QK_SHORT_RI1=0) and the long-chain kernel (QK_SHORT_CHAIN=0) must give
    the same bits — every layout runs the same per-pair recurrence."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    res = {}
    for name, env in (("ri1", {}), ("ri2", {"QK_SHORT_RI1": "0"}),
                      ("long", {"QK_SHORT_CHAIN": "0"})):
        path = str(tmp_path / f"{name}.npz")
        subprocess.run([sys.executable, "-c", _LAYOUT_PROBE.format(root=root, path=path)],
                       check=True, env={**os.environ, **env}, timeout=300)
        with np.load(path) as z:
            res[name] = {k: z[k] for k in z.files}
    for k in res["ri1"]:
        assert np.array_equal(res["ri1"][k], res["ri2"][k]), k
        assert np.array_equal(res["ri1"][k], res["long"][k]), k
