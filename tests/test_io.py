"""Matrix Market + layout + rhs ingestion (matrix_io.cpp,
ingest_external harness.cpp:153-188) and acceptance criterion 11 (export /
ingest round trip with identical iterations and bitwise-identical x)."""
import numpy as np
import pytest

from paper_1912_04385_b200.api import IoError
from tests.systems import small_system


@pytest.fixture(params=["orc", pytest.param("gpu", marks=pytest.mark.gpu)])
def api(request):
    return request.getfixturevalue(request.param)


def write_reference_format(a, b, base, drop_layout_t=False):
    """write_block_matrix + write_vector with the reference's formats."""
    nb, n = a.nb, a.dim
    blocks = a.blocks()
    lines = []
    for c in range(a.n_cells):
        for r in range(nb):
            for k in range(a.row_ptr[c], a.row_ptr[c + 1]):
                for q in range(nb):
                    lines.append("%d %d %.17g" % (c * nb + r + 1, a.col_idx[k] * nb + q + 1, blocks[k][r][q]))
    with open(base + ".mtx", "w") as f:
        f.write("%%%%MatrixMarket matrix coordinate real general\n%d %d %d\n" % (n, n, len(lines)))
        f.write("\n".join(lines) + "\n")
    with open(base + ".layout", "w") as f:
        f.write("%d %d\n" % (n, a.n_cells))
        for c in range(a.n_cells):
            for r in range(nb):
                tag = "s" if r < nb - 2 else ("P" if r == nb - 2 else "T")
                if drop_layout_t and c == 1 and tag == "T":
                    tag = "s"
                f.write("%d %s\n" % (c, tag))
    with open(base + ".rhs", "w") as f:
        f.write("\n".join("%.17g" % x for x in b) + "\n")


def test_ingest_reproduces_the_system_bitwise(api, tmp_path):
    a, b, _ = small_system("g12x10_nb4_band")
    base = str(tmp_path / "sys")
    write_reference_format(a, b, base)
    s = api.ingest(base + ".mtx", base + ".layout", base + ".rhs")
    assert np.array_equal(s.a.row_ptr, a.row_ptr) and np.array_equal(s.a.col_idx, a.col_idx)
    assert np.array_equal(s.a.values, a.values)
    assert np.array_equal(s.b, b)


def test_ingest_rejects_missing_temperature(api, tmp_path):
    a, b, _ = small_system("g8x6_nb3")
    base = str(tmp_path / "bad")
    write_reference_format(a, b, base, drop_layout_t=True)
    with pytest.raises(IoError):
        api.ingest(base + ".mtx", base + ".layout", base + ".rhs")


def test_ingest_rejects_bad_header_and_rhs(api, tmp_path):
    a, b, _ = small_system("g8x6_nb3")
    base = str(tmp_path / "s")
    write_reference_format(a, b, base)
    with open(base + ".rhs", "w") as f:
        f.write("1.0\n2.0\n")
    with pytest.raises(IoError):
        api.ingest(base + ".mtx", base + ".layout", base + ".rhs")
    write_reference_format(a, b, base)
    with open(base + ".mtx") as f:
        txt = f.read().replace("general", "symmetric", 1)
    with open(base + ".mtx", "w") as f:
        f.write(txt)
    with pytest.raises(IoError):
        api.ingest(base + ".mtx", base + ".layout", base + ".rhs")


def test_duplicates_are_summed_and_zero_diagonal_blocks_inserted(orc, tmp_path):
    """from_triplets sums duplicates; assemble inserts missing diagonal blocks."""
    base = str(tmp_path / "d")
    with open(base + ".mtx", "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n% comment\n4 4 4\n1 1 2.0\n1 1 0.5\n1 3 1.0\n3 3 4.0\n")
    with open(base + ".layout", "w") as f:
        f.write("4 2\n0 P\n0 T\n1 P\n1 T\n")
    with open(base + ".rhs", "w") as f:
        f.write("1\n2\n3\n4\n")
    s = orc.ingest(base + ".mtx", base + ".layout", base + ".rhs")
    assert list(s.a.row_ptr) == [0, 2, 3] and list(s.a.col_idx) == [0, 1, 1]
    blocks = s.a.blocks()
    assert blocks[0][0][0] == 2.5 and blocks[1][0][0] == 1.0 and blocks[2][0][0] == 4.0


@pytest.mark.gpu
def test_acceptance_11_gpu_roundtrip_identical_solution(gpu, orc, tmp_path):
    """GPU writer -> GPU and oracle ingestion bitwise; the ingested system solves to
    the same iterations and bitwise-identical x (acceptance.cpp:408-425)."""
    a, b, _ = small_system("g16x16_nb8_band")
    base = str(tmp_path / "rt")
    direct = gpu.system(a).setup("cptr3-amg", b)
    r0 = direct.solve()
    direct.write(base + ".mtx", base + ".layout", base + ".rhs")
    sg = gpu.ingest(base + ".mtx", base + ".layout", base + ".rhs")
    so = orc.ingest(base + ".mtx", base + ".layout", base + ".rhs")
    assert np.array_equal(sg.a.values, a.values) and np.array_equal(so.a.values, a.values)
    assert np.array_equal(sg.b, b)
    r1 = sg.setup("cptr3-amg").solve()
    assert r1.iterations == r0.iterations
    assert np.array_equal(r1.x, r0.x)
