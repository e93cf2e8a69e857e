"""The product's task feeder (csrc/tasks.cu: generate_instance / reward, tasks.cpp:105-175)
against the unmodified reference (oracle/_ref) on CPU: prompts, answers and rewards
bit-identical for every task kind, both vocabularies, many seeds; expert traces (always
reward 1 in the reference) and random / corrupted completions."""
import ctypes as C

import numpy as np
import pytest

import oracle_ffi as O
import paper_2505_17218_b200 as D

pytestmark = pytest.mark.ref
KINDS = [D.TASK_ADD, D.TASK_MOD, D.TASK_REVERSE, D.TASK_PARITY, D.TASK_MICRO]


def ref_fns():
    R = O.ref()
    R.ref_task_instance.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, O.i32p, O.i32p, C.c_char_p, C.c_int]
    R.ref_task_reward.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, O.i32p, C.c_int, O.f64p]
    R.ref_task_expert.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, O.i32p, C.c_int, O.i32p]
    return R


@pytest.mark.parametrize("vocab", [D.VOCAB_TASK, D.VOCAB_BYTE])
@pytest.mark.parametrize("kind", KINDS)
def test_instances_match_reference(kind, vocab):
    R = ref_fns()
    for difficulty in (1, 2, 3, 5):
        seeds = [O.derive_seed(7, "prompt", m, difficulty) for m in range(200)] + [0, 1, 2 ** 64 - 1]
        toks, off, answers = D.task_instances(kind, difficulty, seeds, vocab)
        for i, sd in enumerate(seeds):
            pr = np.zeros(64, dtype=np.int32)
            m = C.c_int32(0)
            ans = C.create_string_buffer(64)
            assert R.ref_task_instance(kind, difficulty, vocab, sd, O.ptr(pr, O.i32p), C.byref(m), ans, 64) == 0
            assert np.array_equal(toks[off[i]:off[i + 1]], pr[:m.value]), (kind, difficulty, sd)
            assert answers[i] == ans.value.decode()


@pytest.mark.parametrize("vocab", [D.VOCAB_TASK, D.VOCAB_BYTE])
@pytest.mark.parametrize("kind", KINDS)
def test_rewards_match_reference(kind, vocab):
    R = ref_fns()
    rng = np.random.default_rng(kind * 2 + vocab)
    V = D.task_vocab_size(kind, vocab)
    delim = ord("#") if vocab == D.VOCAB_BYTE else None
    for difficulty in (1, 2, 4):
        seeds = [O.derive_seed(3, "prompt", m, difficulty) for m in range(40)]
        G, ML = 4, 48
        comps = np.full((len(seeds) * G, ML), -1, dtype=np.int32)
        lens = np.zeros(len(seeds) * G, dtype=np.int32)
        for m, sd in enumerate(seeds):
            for g in range(G):
                s = m * G + g
                c = np.zeros(ML, dtype=np.int32)
                n = C.c_int32(0)
                if g < 2:   # expert trace (terse / stepwise): reward 1 in the reference
                    assert R.ref_task_expert(kind, difficulty, vocab, sd, g, O.ptr(c, O.i32p), ML, C.byref(n)) == 0
                    L = n.value
                    if g == 1 and L > 2 and rng.random() < 0.5:   # corrupt one answer token
                        c[L - 2] = int(rng.integers(2, V))
                else:       # random ids, sometimes with delimiters / EOS / spaces
                    L = int(rng.integers(0, ML))
                    c[:L] = rng.integers(1, V, size=L)
                    if L and delim is not None and rng.random() < 0.5:
                        c[int(rng.integers(0, L))] = delim
                comps[s, :L] = c[:L]
                lens[s] = L
        got = D.task_rewards(kind, difficulty, seeds, G, comps, lens, vocab)
        for s in range(len(seeds) * G):
            r = C.c_double(0)
            assert R.ref_task_reward(kind, difficulty, vocab, seeds[s // G], O.ptr(np.ascontiguousarray(comps[s]),
                                     O.i32p), int(lens[s]), C.byref(r)) == 0
            assert got[s] == r.value, (kind, difficulty, s)
        assert got.reshape(-1, G)[:, 0].min() == 1.0      # expert traces always score


def test_task_errors():
    with pytest.raises(D.InputError):
        D.task_instances(D.TASK_ADD, 0, [1])
    with pytest.raises(D.InputError):
        D.task_instances(9, 1, [1])
    assert D.task_vocab_size(D.TASK_ADD) == 16 and D.task_vocab_size(D.TASK_ADD, D.VOCAB_BYTE) == 256
    toks, off, ans = D.task_instances(D.TASK_ADD, 2, [12345], D.VOCAB_BYTE)
    assert "".join(chr(t) for t in toks[1:]) == "76+51=" and ans == ["127"]
