"""§8(f) rows 3-4 pinned to the reference itself (oracle/_ref, built from the
unmodified /root/reference sources):

* the tuning documents this repository writes (api.tuning_result_to_json,
  the committed GPU sweeps in tuning/) are read by the reference's own
  tuning_result_from_json (report_io.cpp:106-157) with the same records,
  best index and best configuration, and the reference's re-serialisation
  (tuning_result_to_json, report_io.cpp:58-102) is the same document minus
  the GPU knobs ("b200" objects, which its reader ignores);
* the SIGPROC transpose the device kernel implements is checked against the
  reference's parse_sigproc (sigproc.cpp:83-191) here, on CPU, so the GPU
  test (test_gpu_parity.py::test_sigproc_transpose_matches_reference) can use
  the same reference parse as its checker.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _need_ref():
    if O.ref_lib() is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")


def _strip_gpu(doc):
    doc = json.loads(json.dumps(doc))
    doc.pop("b200", None)  # sweep-level GPU metadata (tune.py)
    for r in doc["records"]:
        r.pop("b200", None)
    return doc


@pytest.mark.parametrize("name", ["apertif_2", "apertif_4096", "lofar_64", "lofar_4096"])
def test_reference_reads_our_tuning_documents(name):
    _need_ref()
    text = open(os.path.join(ROOT, "tuning", f"{name}.json")).read()
    ref = O.ref_tuning_roundtrip(text)
    if ref is None:
        pytest.skip("oracle/_ref built without json.hpp")
    ours = json.loads(text)
    best = ours["records"][ours["best_index"]]
    assert ref["records"] == len(ours["records"])
    assert ref["best_index"] == ours["best_index"]
    assert ref["num_dms"] == ours["num_dms"]
    assert ref["best_config"] == (best["items_time"], best["items_dm"], best["work_time"],
                                  best["work_dm"])
    assert ref["best_gflops"] == best["gflops"]
    # the reference's own document is ours without the GPU knobs, key for key
    assert json.loads(ref["json"]) == _strip_gpu(ours)


def test_our_reader_takes_the_reference_document():
    """The reference's serialisation (no "b200" objects) loads in api with
    default GPU knobs, and the result writes back to the same document."""
    _need_ref()
    from paper_1601_05052_b200 import api
    text = open(os.path.join(ROOT, "tuning", "lofar_8.json")).read()
    ref = O.ref_tuning_roundtrip(text)
    if ref is None:
        pytest.skip("oracle/_ref built without json.hpp")
    res = api.tuning_result_from_json(ref["json"])
    assert all(r.staging == "auto" and r.flags == 0 for r in res.records)
    back = json.loads(api.tuning_result_to_json(res))
    assert _strip_gpu(back) == json.loads(ref["json"])


def test_runs_are_recorded_in_new_documents():
    """Every timed run rides in runs_s (report_io.cpp:70-79) for sweeps made
    with the round-2 tuner (older committed sweeps predate it)."""
    docs = [json.load(open(p)) for p in glob.glob(os.path.join(ROOT, "tuning", "*_*.json"))
            if not p.endswith("_summary.json")]
    fresh = [d for d in docs if d.get("b200", {}).get("l2") == "flushed"]
    for d in fresh:
        assert all(len(r["runs_s"]) == d["repeats"] for r in d["records"])


@pytest.mark.parametrize("t,c", [(1, 1), (7, 3), (1001, 37), (64, 256)])
def test_sigproc_transpose_restatement_matches_reference(t, c):
    """The restatement the GPU test also relies on: payload[j][k] (time-major,
    k = 0 the highest channel) lands at [c-1-k][j] -- checked against the
    reference's parse_sigproc, including the byte offset of the first
    non-finite sample it rejects."""
    _need_ref()
    rng = np.random.default_rng(t * 1000 + c)
    payload = rng.standard_normal((t, c)).astype(np.float32)
    stream = O.sigproc_bytes(payload, 2000, 1500.0, -0.5)
    out, (f_min, width, rate) = O.ref_parse_sigproc(stream)
    assert np.array_equal(out.view(np.uint32), payload[:, ::-1].T.copy().view(np.uint32))
    assert (f_min, width, rate) == (1500.0 + (c - 1) * -0.5, 0.5, 2000)
    header_end = len(stream) - payload.nbytes
    if t * c > 2:
        j, k = (t * c // 2) // c, (t * c // 2) % c
        payload[j, k] = np.inf
        payload[-1, -1] = np.nan
        bad, offset = O.ref_parse_sigproc(O.sigproc_bytes(payload, 2000, 1500.0, -0.5))
        assert bad is None and offset == header_end + 4 * (j * c + k)
