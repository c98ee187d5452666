"""CGS1 model IO (reference modelio.py:58-127) against the reference's own bytes
(tests/golden/modelio.npz, made by tests/golden/make_golden.py modelio)."""

import numpy as np
import pytest

from conftest import golden

torch = pytest.importorskip("torch")


def test_corrupt_files_raise_reference_errors():
    """Parsing errors happen before any device allocation: CPU-testable."""
    from paper_2509_03775_b200 import modelio
    d = golden("modelio")
    for name in d["bad"]:
        blob = d[f"bad_{name}_bytes"].tobytes()
        with pytest.raises(modelio.ModelFormatError) as e:
            modelio.deserialize_model(blob)
        assert str(e.value) == str(d[f"bad_{name}_msg"])


def test_metrics_csv_schema(tmp_path):
    from paper_2509_03775_b200 import modelio
    from paper_2509_03775_b200.sampler import TransitionRecord
    recs = [TransitionRecord(iteration=1, kind="update", codebook="-", attempts=1, accepts=1,
                             live_sh=3, live_sr=4, recon=0.25),
            TransitionRecord(iteration=2, kind="split", codebook="sh", attempts=5, accepts=0,
                             live_sh=3, live_sr=4)]
    p = tmp_path / "m.csv"
    modelio.write_metrics_csv(recs, p)
    lines = p.read_text().splitlines()
    assert lines[0] == modelio.CSV_HEADER
    assert lines[1].startswith("1,update,-,1,1,3,4,0.25,")
    assert lines[2].split(",")[7] == "nan"


@pytest.mark.gpu
def test_serialize_matches_reference_bytes():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from gpu_helpers import state_from
    from paper_2509_03775_b200 import modelio
    d = golden("modelio")
    m = golden("mcmc")
    for case in d["cases"]:
        st = state_from(m, str(case) + "_")
        ref = d[f"{case}_bytes"].tobytes()
        data = modelio.serialize_model(st)
        assert data == ref, case
        # round trip: load on the device, serialise again
        st2 = modelio.deserialize_model(data)
        assert modelio.serialize_model(st2) == ref
        assert st2.sh.live_count == st.sh.live_count and st2.sr.live_count == st.sr.live_count
