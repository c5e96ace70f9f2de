"""On-disk inputs: PFMC1 checkpoints and PSEQ1 sequence files written by the unmodified reference
(tests/golden/files.npz, make_golden.py:gen_files) read back by the package, written back byte
for byte, and scored. Mirrors test_model.cpp:564-606 and test_seqdata.cpp:167-227."""
import numpy as np
import pytest

import golden_util as G
from oracle import pyoracle
from paper_2507_12704_b200 import ckpt, seqfile
from paper_2507_12704_b200.abi import FinetuneSpec


@pytest.fixture(scope="module")
def orc():
    return pyoracle.oracle()


@pytest.mark.parametrize("name", ["ckpt_learned", "ckpt_nopos"])
def test_checkpoint_roundtrip(orc, name):
    z = G.load("files")
    raw = z[name + ".file"].tobytes()
    _, w = G.weights_from(z, orc, name + ".")
    ck = ckpt.loads_checkpoint(raw)
    assert ck.spec == w.spec
    for a, b in zip(ck.tensors, w.tensors):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ck.table, w.table)
    np.testing.assert_array_equal(ck.table_seeds, w.table_seeds)
    assert "run.note=golden" in ck.config_text
    with_head = name == "ckpt_learned"
    if with_head:
        h = ck.head()
        for k in ("d_module", "d_emb", "n_ctx", "hidden", "d_aux"):
            assert h[k] == w.head[k], k
        for k in ("w1", "b1", "w2", "b2", "mod_w", "mod_b", "aux_proj", "lt"):
            np.testing.assert_array_equal(h[k].reshape(-1), np.asarray(w.head[k]).reshape(-1), err_msg=k)
    else:
        assert ck.head() is None
        with pytest.raises(ValueError, match="no ranking head"):
            ck.weights()
    # save_checkpoint parity: the package writes the reference's bytes
    assert ckpt.dumps_checkpoint(w, "run.note=golden\n", with_head=with_head) == raw


def test_checkpoint_scores(orc):
    """A model loaded from the reference's checkpoint scores like the model that was saved."""
    z = G.load("files")
    w = ckpt.loads_checkpoint(z["ckpt_learned.file"].tobytes()).weights()
    b = G.batch_from(z, "ckpt_learned.")
    logits = orc.rank_forward_batch(w, FinetuneSpec(max_events=10), b)[0]
    np.testing.assert_array_equal(logits, z["ckpt_learned.logits"])


def test_checkpoint_errors():
    z = G.load("files")
    raw = z["ckpt_learned.file"].tobytes()
    cases = [(b"XFMC1" + raw[5:], "bad checkpoint magic"), (raw[:7], "truncated while reading config length"),
             (raw[:-3], "truncated while reading"), (raw + b"\0", "trailing bytes after checkpoint blobs")]
    for bad, msg in cases:
        with pytest.raises(ValueError, match=msg):
            ckpt.loads_checkpoint(bad)
    nb = ckpt.loads_blobs(raw)
    nb.blobs = [(n, m) for n, m in nb.blobs if n != "layer1.wq"]
    with pytest.raises(ValueError, match="missing parameter blob 'layer1.wq'"):
        ckpt.loads_checkpoint(ckpt.dumps_blobs(nb))
    nb = ckpt.loads_blobs(raw)
    nb.blobs = [(n, m[:, :-1] if n == "phi_out.w2" else m) for n, m in nb.blobs]
    with pytest.raises(ValueError, match="'phi_out.w2' has shape 16x15, expected 16x16"):
        ckpt.loads_checkpoint(ckpt.dumps_blobs(nb))
    with pytest.raises(ValueError, match="config line 1 is not key=value"):
        ckpt.parse_kv_text("no equals sign\n")


def test_sequences_roundtrip():
    z = G.load("files")
    raw = z["seq.file"].tobytes()
    s = seqfile.loads(raw)
    for k in ("user_ids", "offsets", "ts", "action", "surface", "item"):
        np.testing.assert_array_equal(getattr(s, k), z["seq." + k], err_msg=k)
    assert s.config_text == "data.seed=31\n"
    assert seqfile.dumps(s) == raw


def test_sequences_errors():
    z = G.load("files")
    raw = bytearray(z["seq.file"].tobytes())
    hdr = 5 + 4 + 8 + 4  # magic, user count, first user's id and event count
    bad_action = bytearray(raw)
    bad_action[hdr + 8] = 9  # first record's action
    bad_ts = bytearray(raw)
    bad_ts[hdr + 18:hdr + 26] = (0).to_bytes(8, "little")  # second record's timestamp < first
    for bad, msg in ((b"XSEQ1" + bytes(raw[5:]), "bad magic"), (bytes(raw[:7]), "too short for header"),
                     (bytes(bad_action), "invalid action value 9 at record 0"),
                     (bytes(bad_ts), "non-monotonic timestamp at record 1"),
                     (bytes(raw[:hdr + 10]), "truncated while reading"),
                     (bytes(raw) + b"\0", "trailing bytes after config trailer")):
        with pytest.raises(ValueError, match=msg):
            seqfile.loads(bad)


def test_ranking_batch_from_sequences(orc):
    """Scoring a PSEQ1 dataset: rows of one user share the newest max_events events; the
    oracle's plan dedups them to one unique per user with events."""
    z = G.load("files")
    s = seqfile.loads(z["seq.file"].tobytes())
    users = [0, 2, 2, 3, 4, 0]
    b = seqfile.ranking_batch(s, users, candidates=[11, 12, 13, 14, 15, 16], ages=[3600.0] * 6, max_events=6)
    assert list(b.row_valid) == [5, 6, 6, 1, 6, 5]
    np.testing.assert_array_equal(b.row_offset[1:3], [s.offsets[3] - 6] * 2)
    rep, first, b_u = orc.dedup(b)
    assert b_u == 4
