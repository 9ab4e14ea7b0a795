"""Pins for the shared input generators (kvgen): published vectors and stated distributions."""
import numpy as np

from kvgen import configs
from kvgen.content import (GOLDEN, content_keys, content_segment_table, content_tokens,
                           splitmix64, splitmix64_int)
from kvgen.schedule import closed_loop_schedule
from kvgen.trace import poisson_arrivals, synth_trace


def test_splitmix64_published_vectors():
    # Steele, Lea & Flood SplitMix64; state 0 -> first output 0xE220A8397B1DCDAF, and the
    # widely published sequence for seed 1234567 (outputs 1..5).
    assert splitmix64_int(0) == 0xE220A8397B1DCDAF
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423,
            4593380528125082431, 16408922859458223821]
    got = [splitmix64_int((1234567 + k * GOLDEN) % 2**64) for k in range(5)]
    assert got == want
    vec = splitmix64(np.array([(1234567 + k * GOLDEN) % 2**64 for k in range(5)], dtype=np.uint64))
    assert [int(x) for x in vec] == want


def test_content_closed_form_structure():
    L, H, d = 2, 8, 128
    t = content_segment_table(2601, 4, L, H, d)
    x = content_tokens(2601, [7, 7, 9], [0, 1, 0], 4, L, H, d)
    k = content_keys(2601, [7, 7, 9], [0, 1, 0])
    for n in range(3):
        for dim in (0, 1, 2, 3, 77):
            w = (int(k[n]) >> (16 * (dim % 4))) & 0xFFFF
            assert x[n, 1, 0, 3, dim] == t[1, 0, 3, dim] ^ w
    # the table is a function of the GLOBAL layer: stage 2 layer 0 == layer 4
    t_all = content_segment_table(2601, 0, 8, H, d)
    assert np.array_equal(t_all[4:6], t)


def test_content_segments_distinct():
    # a misplaced 256-B segment must always be detectable: all segments of a sample differ
    x = content_tokens(2601, np.repeat(np.arange(8), 16), np.tile(np.arange(16), 8), 0, 8, 8, 128)
    segs = x.reshape(-1, 128)
    assert len({s.tobytes() for s in segs}) == segs.shape[0]


def test_trace_shape_spec_s466():
    p, o = synth_trace(10000, 22438)
    assert p.min() >= 1 and p.max() <= 2048 and o.min() >= 1 and o.max() <= 1024
    assert 115 <= np.median(p) <= 141          # median prompt within +-10 % of 128
    assert 115 <= np.median(o) <= 141
    p2, _ = synth_trace(10000, 22438)
    assert np.array_equal(p, p2)


def test_poisson_mean_count_spec_s462():
    counts = [np.sum(poisson_arrivals(2.0, 2000, s) <= 600.0) for s in range(200)]
    assert abs(np.mean(counts) - 1200) < 3 * np.sqrt(1200)
    assert poisson_arrivals(0, 10, 1).size == 0


def test_closed_loop_schedule_semantics():
    sch = closed_loop_schedule([5, 3, 7], [2, 1, 3], n_steps=8, cap=2)
    ev = sch.steps
    assert ev[0].admit == [(0, 5), (1, 3)] and ev[0].decode == []
    assert ev[1].decode == [0, 1]
    # request 1 (O=1): last token at step 1 -> retires at step 2; request 2 admitted then
    assert ev[2].retire == [1] and ev[2].admit == [(2, 7)] and ev[2].decode == [0]
    assert ev[3].retire == [0]
    assert sch.length_at(0, 2) == 7 and sch.length_at(2, 5) == 10
    for r, req in sch.requests.items():
        assert sum(r in e.decode for e in ev) == req.output


def test_c1_schedule():
    (sch,) = configs.build_schedules(configs.C1)
    assert sch.steps[0].admit == [(0, 64), (1, 64), (2, 64), (3, 64)]
    for t in range(1, 9):
        assert sch.steps[t].decode == [0, 1, 2, 3] and not sch.steps[t].admit
