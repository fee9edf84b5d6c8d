"""Shard layer on the GPU: record-range shards of a C3-like batch, each
validated through the batch entry point (one after another on one GPU),
concatenate to the whole batch's verdicts and to the oracle's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_record_shards_on_gpu_match_whole_batch():
    import paper_2010_03090_b200 as u8
    from paper_2010_03090_b200 import configs, sharding
    b = configs.gen_c3(n_records=20000, seed=9)
    data = b.data.cpu().numpy()
    offs = b.offsets if hasattr(b, "offsets") else b.d_offsets.cpu().numpy()
    whole = u8.validate_lookup_batch(data, offs)
    assert (whole == b.expected).all()
    for world in (1, 2, 3, 8):
        shards = sharding.plan_records(offs, world)
        parts = [sharding.validate_batch_sharded(data, offs, sh) for sh in shards]
        assert (np.concatenate(parts) == whole).all(), world
