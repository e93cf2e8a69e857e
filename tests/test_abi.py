"""CPU-side checks of the drop-in boundary: libdashcu.so loads, exports every
symbol include/dashcu.h declares, host-only entry points agree with the oracle,
and compute entry points fail loudly (no CPU fallback) when no B200 is visible."""
import ctypes as C
import os
import re

import pytest

import oracle_ffi as O
import paper_2505_17218_b200 as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dashcu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:DASHCU_API\s+)?(?:const char\*|int64_t|int)\s+(dashcu_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("dashcu_sample", "dashcu_advantage_filter", "dashcu_accumulate", "dashcu_optimizer_step",
                 "dashcu_allreduce_grads", "dashcu_rollout_log_prob", "dashcu_policy_upload"):
        assert must in syms
    assert len(syms) >= 30


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(D.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_num_params_matches_oracle():
    for arch in (dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0, eos_id=1),
                 dict(vocab_size=151936, embed_dim=896, context_len=1152, ffn_hidden=4864, n_layers=24, bos_id=0,
                      eos_id=1, n_heads=14, n_kv_heads=2, head_dim=64)):
        assert D.num_params(arch) == O.num_params(arch)
    assert D.num_params(dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0,
                             eos_id=1)) == 468480


def test_arch_validation_errors():
    with pytest.raises(D.InputError):
        D.num_params(dict(vocab_size=2, embed_dim=4, context_len=8, ffn_hidden=4, n_layers=1, bos_id=-1, eos_id=1))
    with pytest.raises(D.InputError):
        D.num_params(dict(vocab_size=8, embed_dim=4, context_len=8, ffn_hidden=4, n_layers=1, bos_id=1, eos_id=1))
    with pytest.raises(D.InputError):
        D.num_params(dict(vocab_size=8, embed_dim=4, context_len=8, ffn_hidden=4, n_layers=1, bos_id=0, eos_id=1,
                          n_heads=3, n_kv_heads=2, head_dim=2))


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is visible")
    with pytest.raises(D.DeviceError):
        D.Context(0)


def test_shard_span_partitions_the_flat_vector():
    """dashcu_shard_span (the sharded optimizer's slices): disjoint, ordered, covering,
    64-element aligned, equal slice strides (in-place reduce-scatter / all-gather)."""
    for total in (1, 63, 64, 65, 468480, 527_000_123):
        for world in (1, 2, 3, 4, 7, 8):
            spans = [D.shard_span(total, world, r) for r in range(world)]
            stride = ((total + world - 1) // world + 63) // 64 * 64
            pos = 0
            for r, (off, n) in enumerate(spans):
                assert off == r * stride and off % 64 == 0 and 0 <= n <= stride
                if n:
                    assert off == pos
                    pos += n
            assert pos == total
    with pytest.raises(D.InputError):
        D.shard_span(10, 2, 2)
