"""a partitioned index (each part keeps the SA ranks and table entries of one route-key
range).  Routing + per-part search + scatter must reproduce the replicated index's intervals exactly; the
exchange is emulated in-process here (tests/test_dist_gloo.py and the 2-rank bench run cover the
collective path)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
import paper_1303_3692_b200 as sa  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", ["rec32", "rec16", "plain"])
@pytest.mark.parametrize("nparts", [2, 3, 7])
def test_partitions_reproduce_replicated(layout, nparts):
    ref = synth.reference(synth.REF_REPEAT, 2_000_000, 91)
    words, lens = synth.reads(ref, 60_000, 16, 140, 0.1, 0.01, 92)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = torch.from_numpy(lens.view(np.int32)).cuda()
    full = sa.Index(ref, layout=layout)
    want = full.match(w, l)
    parts = [sa.Index(ref, layout=layout, part=(g, nparts, 8)) for g in range(nparts)]
    infos = [p.part_info() for p in parts]
    assert infos[0]["rank_lo"] == 0 and infos[-1]["rank_hi"] == len(ref)
    for a, b in zip(infos, infos[1:]):
        assert a["rank_hi"] == b["rank_lo"]          # the slices tile the SA
    order, ow, ol, offs = parts[0].route(w, l)
    offs = offs.cpu().tolist()
    assert offs[0] == 0 and offs[-1] == 60_000
    res = torch.empty_like(want)
    for g in range(nparts):
        if offs[g + 1] > offs[g]:
            res[offs[g]:offs[g + 1]] = parts[g].match(ow[offs[g]:offs[g + 1]], ol[offs[g]:offs[g + 1]])
    got = sa.scatter_results(order, res)
    assert torch.equal(got, want)


def test_partition_rejects_short_reads():
    ref = synth.reference(synth.REF_UNIFORM, 300_000, 5)
    part = sa.Index(ref, part=(0, 2, 4))
    words, lens = synth.pack_strings(["ACGT", "A" * 40])
    got = part.match(torch.from_numpy(words.view(np.int64)).cuda(), torch.from_numpy(lens.view(np.int32)).cuda())
    got = got.cpu().numpy().view(np.uint32)
    assert got[0].tolist() == [0xFFFFFFFF, 0xFFFFFFFF]
