"""Wire format (paper_2412_15126_b200/wire.py): round trips on the CPU oracle
engine, parameter checks, and (GPU) bit-exact interchange between the B200
engine and the oracle engine."""
import numpy as np
import pytest

from oracle.oracle import oracle_engine
from paper_2412_15126_b200 import wire
from paper_2412_15126_b200.engine import IncompatibleParamsError
from paper_2412_15126_b200.keys import sample_secret
from paper_2412_15126_b200.params import preset


def test_ciphertext_roundtrip_oracle(tmp_path):
    eng = oracle_engine(preset("toy"))
    v = np.linspace(-0.5, 0.5, 16)
    ct = eng.rotate(eng.encrypt(v), 3)
    path = tmp_path / "ct.npz"
    wire.save_ciphertext(path, eng, ct)
    back = wire.load_ciphertext(path, eng)
    assert back.level == ct.level and back.rot_chain == ct.rot_chain
    assert np.array_equal(np.asarray(back.data), np.asarray(ct.data))
    assert np.allclose(eng.decrypt(back)[:16], np.concatenate([v[3:], np.zeros(3)]), atol=1e-6)


def test_params_mismatch_and_bad_files(tmp_path):
    a, b = oracle_engine(preset("toy")), oracle_engine(preset("toy_deep"))
    path = tmp_path / "ct.npz"
    wire.save_ciphertext(path, a, a.encrypt([0.25, 0.5]))
    with pytest.raises(IncompatibleParamsError):
        wire.load_ciphertext(path, b)
    sk = tmp_path / "sk.npz"
    wire.save_secret(sk, a, sample_secret(a.params))
    with pytest.raises(ValueError):
        wire.load_ciphertext(sk, a)  # a secret file is not a ciphertext
    with pytest.raises(ValueError):
        wire.save_secret(sk, a, np.full(a.params.ring_degree, 2))


def test_secret_roundtrip_regenerates_keys(tmp_path):
    p = preset("toy")
    a, b = oracle_engine(p), oracle_engine(p)
    s = sample_secret(p)
    s2 = s.copy()
    s2[:2] = -s2[:2] if np.any(s2[:2]) else [1, -1]
    b.use_secret(s2)  # b now decrypts nothing of a's ...
    path = tmp_path / "sk.npz"
    wire.save_secret(path, a, s)
    b.use_secret(wire.load_secret(path, b))  # ... until it loads a's secret
    v = np.array([0.1, 0.7, 0.3])
    ct_a = a.rotate(a.encrypt(v), 1)
    ct_b = b.rotate(b.encrypt(v), 1)
    assert np.array_equal(np.asarray(ct_a.data), np.asarray(ct_b.data))


@pytest.mark.gpu
def test_gpu_oracle_interchange(tmp_path, require_cuda):
    from paper_2412_15126_b200 import B200Engine

    p = preset("toy_deep")
    gpu, cpu = B200Engine(p), oracle_engine(p)
    v = np.array([0.30, 0.10, 0.80, 0.55, 0.20, 0.95, 0.65, 0.40])
    path = tmp_path / "x.npz"
    # GPU -> oracle: the GPU product, checked on the oracle
    xg = gpu.encrypt(v)
    wire.save_ciphertext(path, gpu, xg)
    xc = wire.load_ciphertext(path, cpu)
    mg, mc = gpu.mul(gpu.rotate(xg, 5), xg), cpu.mul(cpu.rotate(xc, 5), xc)
    wire.save_ciphertext(path, gpu, mg)
    assert np.array_equal(wire.load_ciphertext(path, cpu).data, mc.data)
    # oracle -> GPU
    wire.save_ciphertext(path, cpu, mc)
    back = wire.load_ciphertext(path, gpu)
    assert np.array_equal(gpu.backend.to_host(back.data), mc.data)
    assert np.allclose(gpu.decrypt(back)[:8], np.concatenate([v[5:] * v[:3], np.zeros(5)]), atol=1e-5)
