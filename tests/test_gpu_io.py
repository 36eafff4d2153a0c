"""GPU: pipelined campaign (F3) against the staged path + reference file format, and device stats (F4)."""
import json
import zlib
from pathlib import Path

import numpy as np
import pytest

import parity
from paper_2205_07976_b200 import BackgroundProfile, PixelBuffer, simulate_image, synthetic
from paper_2205_07976_b200 import io as nio

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"

WATER = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.162, 8.0), (0.3, 6.5)))


def ctx_for(i, compute="fp32"):
    panel = synthetic.roi(synthetic.rayonix_panel(), 1700, 1800, 96, 128)
    return synthetic.ls49_context(synthetic.SEED + i, panel=panel, n_channels=10, n_domains=4, compute=compute)


@pytest.mark.parametrize("compute", ["fp32", "fp64"])
def test_campaign_files_equal_simulate_image_downcast(gpu, tmp_path, compute):
    res = nio.run_campaign(lambda i: ctx_for(i, compute), 5, tmp_path, first_image=10, background=WATER,
                           thickness_factor=0.5, seeds=lambda i: synthetic.SEED + i)
    assert res.indices == list(range(10, 15))
    for idx, path, crc in zip(res.indices, res.paths, res.crcs):
        data, side = nio.read_image(path)
        assert side["crc32"] == crc == zlib.crc32(path.read_bytes())
        assert side["image_index"] == idx and side["seed"] == synthetic.SEED + idx
        assert side["dims"] == [96, 128] and side["dtype"] == "float32"
        acc = simulate_image(ctx_for(idx, compute), background=WATER, thickness_factor=0.5)
        assert np.array_equal(data.reshape(-1), acc.data.astype(np.float32))


def hot_ctx_for(i, bad=(12,)):
    """Image ``i`` of a campaign whose images in ``bad`` overflow float32 (fluence x 1e40)."""
    import dataclasses

    c = ctx_for(i, "fp64")
    if i in bad:
        c = dataclasses.replace(c, spectrum=dataclasses.replace(c.spectrum, fluence=c.spectrum.fluence * 1e40))
    return c


def test_campaign_flags_faulting_images_and_continues(gpu, tmp_path):
    """A non-finite image is flagged (index, lowest bad pixel) and skipped; the images before and
    after it are written with their sidecars -- the reference's rank loop (scheduler.py:208-214)."""
    from paper_2205_07976_b200 import PatternFault, nanobragg_spots

    res = nio.run_campaign(hot_ctx_for, 5, tmp_path, first_image=10, seeds=lambda i: synthetic.SEED + i)
    assert res.indices == [10, 11, 13, 14]
    with pytest.raises(PatternFault) as info:  # the pixel the drop-in reports for the same image
        nanobragg_spots(hot_ctx_for(12), PixelBuffer.zeros((96, 128), "f32"))
    assert res.flagged == [(12, info.value.index)]
    assert not (tmp_path / "img_000012.bin").exists() and not (tmp_path / "img_000012.json").exists()
    for idx, path in zip(res.indices, res.paths):
        data, side = nio.read_image(path)
        assert side["image_index"] == idx
        acc = simulate_image(ctx_for(idx, "fp64"))
        assert np.array_equal(data.reshape(-1), acc.data.astype(np.float32))


def test_campaign_io_failure_aborts_after_writing_sidecars(gpu, tmp_path):
    """An unwritable image file raises CampaignIOError(index) (scheduler.py:219-225); every image
    written before it has its sidecar and reads back; the images after it are not rendered."""
    from paper_2205_07976_b200.errors import CampaignIOError

    (tmp_path / "img_000013.bin").mkdir()  # fopen(..., "wb") fails on a directory
    with pytest.raises(CampaignIOError) as info:
        nio.run_campaign(lambda i: ctx_for(i, "fp64"), 5, tmp_path, first_image=10)
    assert info.value.image_index == 13 and isinstance(info.value, OSError)
    for idx in (10, 11, 12):
        data, side = nio.read_image(tmp_path / f"img_{idx:06d}.bin")
        assert side["image_index"] == idx
    assert not (tmp_path / "img_000014.bin").exists()


def test_write_image_matches_reference_format(gpu, tmp_path):
    acc = simulate_image(ctx_for(0))
    p = nio.write_image(acc, tmp_path / "x", panel=ctx_for(0).panel, spectrum=ctx_for(0).spectrum, seed=3,
                        image_index=7)
    side = json.loads((tmp_path / "x.json").read_text())
    assert set(side) == {"dims", "dtype", "byte_order", "downcast", "pixel_size_m", "distance_m",
                         "wavelengths_angstrom", "seed", "image_index", "crc32"}
    data, _ = nio.read_image(p)
    assert np.array_equal(data.reshape(-1), acc.data.astype("<f4"))


def reference_stats_total(values: np.ndarray) -> float:
    """The reference's image_stats total restated with NumPy (kernels.py:346-371): per 8192
    block float(np.sum(chunk, dtype=np.float64)), then parallel_reduce's tree that splits a
    span at the largest power of two strictly below its size (execution.py:227-260)."""
    blocks = [float(np.sum(values[i:i + 8192], dtype=np.float64)) for i in range(0, values.size, 8192)]

    def span(lo, hi):
        if hi - lo == 1:
            return blocks[lo]
        mid = lo + (1 << ((hi - lo - 1).bit_length() - 1))
        return span(lo, mid) + span(mid, hi)

    return span(0, len(blocks))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [15, 8192, 3 * 8192, 1_000_000, 14_745_600])
def test_image_stats_total_is_bitwise_the_reference(gpu, dtype, n):
    """Device image_stats reproduces the reference's FP64 total bit for bit: NumPy's pairwise
    sum inside each block and the fixed block tree (nbx_reduce.cu), on data whose summation
    order matters (lognormal over ~14 decades)."""
    rng = np.random.default_rng(n)
    vals = np.exp(rng.normal(0.0, 8.0, n)).astype(dtype)
    st = nio.image_stats(PixelBuffer((1, n), "f32" if dtype == np.float32 else "f64", vals))
    want = reference_stats_total(vals)
    assert st.total == want, (st.total, want)
    assert st.mean == want / n
    assert st.min == float(vals.min()) and st.max == float(vals.max())


def test_image_stats_matches_reference_fixture(gpu):
    """Against xtrace's own image_stats outputs (tests/golden/stats.npz): every field bitwise."""
    z = np.load(GOLDEN / "stats.npz")
    for n, prec, ref in zip(z["n"], z["precision"], z["ref_stats"]):
        n, prec = int(n), str(prec)
        rng = np.random.default_rng(n)  # tools/make_golden.py:stats_values
        v = np.exp(rng.normal(0.0, 8.0, n)).astype(np.float32 if prec == "f32" else np.float64)
        st = nio.image_stats(PixelBuffer((1, n), prec, v))
        assert tuple(st) == tuple(float(x) for x in ref), (n, prec, tuple(st), ref)


def test_image_stats_and_histogram(gpu):
    rng = np.random.default_rng(17)
    vals = rng.uniform(-1, 1, 1_000_000)
    st = nio.image_stats(PixelBuffer((1000, 1000), "f64", vals))
    assert st.min == vals.min() and st.max == vals.max()
    assert st.total == pytest.approx(float(np.sum(vals)), rel=1e-12)
    assert nio.image_stats(PixelBuffer((2, 2), "f64", [1.0, 2.0, 3.0, 4.0])) == (1.0, 4.0, 2.5, 10.0)
    c = nio.image_stats(PixelBuffer((3, 5), "f32", np.full(15, 7.25)))
    assert c.min == c.max == c.mean == 7.25 and c.total == 7.25 * 15
    # determinism: same bits every call
    assert nio.image_stats(PixelBuffer((1000, 1000), "f64", vals)) == st
    vals = rng.uniform(-0.2, 1.2, 100_000)
    h = nio.image_histogram(PixelBuffer((250, 400), "f64", vals), 64, (0.0, 1.0))
    under, over = int((vals < 0).sum()), int((vals > 1).sum())
    idx = np.clip(np.floor((vals[(vals >= 0) & (vals <= 1)] - 0.0) / (1.0 / 64)).astype(np.int64), 0, 63)
    assert h.counts.tolist() == np.bincount(idx, minlength=64).tolist()
    assert (h.underflow, h.overflow) == (under, over)
    assert h.cumulative.tolist() == np.cumsum(h.counts).tolist()
    edge = nio.image_histogram(PixelBuffer((1, 4), "f64", [1.0] * 4), 4, (0.0, 1.0))
    assert edge.counts.tolist() == [0, 0, 0, 4]


HIST_SPECS = [(1, (0.0, 1.0)), (3, (0.1, 0.7)), (64, (-2.5, 7.25)), (1000, (1e-3, 3.0))]


def hist_values(precision):
    """tools/make_golden.py:hist_values -- seeded values plus every binning edge case."""
    rng = np.random.default_rng(42)
    v = [rng.uniform(-3.0, 8.0, 20000), rng.lognormal(0.0, 1.0, 5000)]
    for n_bins, (lo, hi) in HIST_SPECS:
        w = (hi - lo) / n_bins
        edges = lo + w * np.arange(n_bins + 1)
        v += [edges, np.nextafter(edges, -np.inf), np.nextafter(edges, np.inf), [lo, hi]]
    v.append([np.inf, -np.inf, np.nan, 5e-324, -5e-324, 0.0, -0.0])
    out = np.concatenate([np.asarray(x, dtype=np.float64) for x in v])
    return out.astype(np.float32) if precision == "f32" else out


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_histogram_equals_reference_run(gpu, precision):
    """image_histogram against xtrace.kernels.image_histogram's own output
    (tests/golden/histogram.npz): bin edges, one-ulp neighbours, lo/hi, +-inf, NaN (the
    reference's int64 cast puts it in bin 0), subnormals -- counts, cumulative, under/overflow
    exactly equal."""
    golden = np.load(parity.GOLDEN / "histogram.npz")
    vals = hist_values(precision)
    for n_bins, rng_ in HIST_SPECS:
        h = nio.image_histogram(PixelBuffer((1, vals.size), precision, vals), n_bins, rng_)
        key = f"{precision}_{n_bins}"
        assert np.array_equal(h.counts, golden[key + "_counts"]), key
        assert np.array_equal(h.cumulative, golden[key + "_cumulative"]), key
        assert [h.underflow, h.overflow] == golden[key + "_under_over"].tolist(), key


def stats_special_values():
    """tools/make_golden.py:stats_special_values (non-finite placements across 5 blocks)."""
    rng = np.random.default_rng(3)
    base = rng.uniform(-1.0, 1.0, 5 * 8192 - 100)
    cases = []
    for kind, at in (("nan", 5), ("nan", 20000), ("nan", base.size - 1), ("inf", 9000), ("-inf", 30000),
                     ("nan+inf", (100, 17000)), ("zeros", None)):
        v = base.copy()
        if kind == "nan":
            v[at] = np.nan
        elif kind == "inf":
            v[at] = np.inf
        elif kind == "-inf":
            v[at] = -np.inf
        elif kind == "nan+inf":
            v[at[0]] = np.inf
            v[at[1]] = np.nan
        else:
            v = np.where(np.arange(v.size) % 2 == 0, 0.0, -0.0)
        cases.append(v)
    return cases


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_stats_non_finite_semantics_equal_reference_run(gpu, precision):
    """image_stats with NaN / inf against xtrace.kernels.image_stats's own output
    (tests/golden/stats_special.npz): NumPy's NaN-propagating block min/max, then Python's
    min/max along parallel_reduce's tree (a NaN block survives only as a left operand) --
    min, max, mean, total equal as values (the sign of a zero extremum is not pinned)."""
    golden = np.load(parity.GOLDEN / "stats_special.npz")[precision]
    for i, v in enumerate(stats_special_values()):
        vv = v.astype(np.float32 if precision == "f32" else np.float64)
        st = nio.image_stats(PixelBuffer((1, vv.size), precision, vv))
        got = np.array([st.min, st.max, st.mean, st.total])
        assert np.array_equal(got, golden[i], equal_nan=True), (i, got, golden[i])
