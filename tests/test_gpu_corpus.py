"""GPU corpus backend on the reference's own bench corpus
(gallery.py:186-220, tests/golden/corpus.npz): per matrix and method the
scaling s and the product count are bit-exact with the reference's
cos_sin / pade_cos_sin, and the errors against the double-double values
are no worse than the reference's own (cli.py:128-163)."""
import math
import os

import numpy as np
import pytest

from paper_2010_00465_b200 import corpus


def _load(golden_dir):
    d = np.load(os.path.join(golden_dir, "corpus.npz"))
    mats, off = [], 0
    for n in d["dims"]:
        mats.append(d["data"][off:off + n * n].reshape(n, n))
        off += n * n
    return d, mats, [str(t) for t in d["tags"]]


def test_run_record_layout_matches_reference():
    assert [f.name for f in corpus.fields(corpus.RunRecord)] == [
        "matrix_id", "class_tag", "norm", "method", "rel_err_cos", "rel_err_sin",
        "products", "scaling_s", "wall_time"]


def test_corpus_fixture_decodes(golden_dir):
    d, mats, tags = _load(golden_dir)
    assert len(mats) == 69 and tags.count("overscaling") == 9
    assert all(m.shape[0] == m.shape[1] for m in mats)


@pytest.mark.gpu
def test_corpus_against_reference(cuda, golden_dir, tmp_path):
    d, mats, tags = _load(golden_dir)
    recs = corpus.run_corpus(mats, tags)
    assert len(recs) == 2 * len(mats)

    def ok_err(mine, ref, s):
        """Per matrix: no worse than 10x the reference, up to the doubling
        recursion's conditioning (a base-pair perturbation grows up to ~4x
        per step; 64 u 4^s is the Pade parity bar of test_gpu_parity)."""
        if math.isinf(ref):
            return math.isinf(mine) or mine > 1e-6
        return mine <= 10.0 * ref + max(1e-14, 64 * 2.0 ** -53 * 4.0 ** s)

    ratios = {"taylor": [], "pade": []}
    for i in range(len(mats)):
        t, p = recs[2 * i], recs[2 * i + 1]
        assert (t.method, p.method) == ("taylor", "pade")
        assert t.scaling_s == int(d["t_s"][i]), i
        assert t.products == float(d["t_prod"][i]), i
        assert p.scaling_s == int(d["p_s"][i]), i
        assert abs(p.products - float(d["p_prod"][i])) < 1e-12, i
        for r, key in ((t, "t"), (p, "p")):
            for mine, ref in ((r.rel_err_cos, float(d[key + "_ec"][i])),
                              (r.rel_err_sin, float(d[key + "_es"][i]))):
                assert ok_err(mine, ref, r.scaling_s), (i, r, ref)
                if math.isfinite(mine) and math.isfinite(ref) and min(mine, ref) > 1e-15:
                    ratios[r.method].append(mine / ref)
    # over the corpus: statistically as accurate as the reference
    for method, rs in ratios.items():
        assert len(rs) > 50
        assert float(np.exp(np.mean(np.log(rs)))) <= 2.0, (method, rs)
    out = tmp_path / "bench.csv"
    corpus.write_csv(recs, str(out))
    lines = out.read_text().splitlines()
    assert lines[0].split(",")[0] == "matrix_id" and len(lines) == 1 + len(recs)
    assert "taylor_better" in corpus.summary(recs)
