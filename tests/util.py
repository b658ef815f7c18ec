"""Test helpers: the parity metric of DESIGN.md ("Tolerance") and tensor plumbing."""
import numpy as np

FP32_TOL = 1e-4      # BASELINE.json north_star: fp32 embeddings/gradients, max rel. error 1e-4
TF32_TOL = 1e-2      # ... 1e-2 where a reduced-precision (tf32) projection is on the path


def rel_err(got, ref):
    """max_i |g_i - o_i| / max(|o_i|, rms(o)) -- relative above the RMS, RMS-normalised below
    (near-zero entries from signed cancellation do not fail spuriously)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    if ref.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(ref * ref)))
    denom = np.maximum(np.abs(ref), rms if rms > 0 else 1.0)
    return float(np.max(np.abs(got - ref) / denom))


def rel_err_scale(got, ref):
    """max_i |g_i - o_i| / max_i |o_i| -- the error against the tensor's scale.  The bar for
    bf16 projections against the EXACT product (reading 7b): rounding both operands
    to bf16 (RNE, relative error up to 2^-8) gives every output an error of std ~3e-3 of the
    row RMS, so an elementwise 1e-2 bar is crossed by the input rounding alone on large
    tensors; the kernel's arithmetic itself is pinned at FP32_TOL against the oracle on the
    bf16-rounded inputs."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    if ref.size == 0:
        return 0.0
    m = float(np.max(np.abs(ref)))
    return float(np.max(np.abs(got - ref))) / (m if m > 0 else 1.0)


def assert_close_scale(got, ref, tol, what=""):
    e = rel_err_scale(got, ref)
    assert e <= tol, f"{what}: error / max|ref| {e:.3e} > {tol:.0e}"
    return e


def assert_close(got, ref, tol=FP32_TOL, what=""):
    e = rel_err(got, ref)
    assert e <= tol, f"{what}: rel err {e:.3e} > {tol:.0e}"
    return e


def np_(t):
    return t.detach().cpu().numpy()
