"""Comparison metrics (test-side, global flatten per S:510)."""
import numpy as np
import torch


def rel_l2(ref, test):
    ref = np.asarray(ref, dtype=np.float64).ravel()
    test = np.asarray(test, dtype=np.float64).ravel()
    return float(np.linalg.norm(ref - test) / np.linalg.norm(ref))


def cos_sim(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0 and nb == 0:
        return 1.0
    return float(a @ b / (na * nb))


def rms(x):
    x = np.asarray(x, dtype=np.float64)
    return float(np.sqrt(np.mean(x * x)))


def f64(t):
    """torch (any float dtype, CPU or CUDA) -> numpy float64, exactly."""
    return t.detach().to("cpu", torch.float32).numpy().astype(np.float64)


def round_bf16(x):
    """Round a float64 array to bf16 (RNE) and back, for comparison after identical rounding (A18)."""
    return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(torch.bfloat16).to(torch.float64).numpy()


def round_fp16(x):
    """Round a float64 array to fp16 (RNE) and back (the SAGE_FP16 I/O type)."""
    return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(torch.float16).to(torch.float64).numpy()
