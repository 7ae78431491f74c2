"""The DenseNet121 layer table (paper Table 2) and its CSV reader, pinned
against the reference's shipped data file and parser messages."""
import os

import pytest

from paper_2411_19419_b200.layers import LayerConfig, densenet121_layers, load_layer_table

REF_CSV = "/root/reference/proj/data/densenet121_layers.csv"


def test_generated_table_shape():
    rows = densenet121_layers()
    assert len(rows) == 123
    assert rows[0] == LayerConfig("conv0", 224, 224, 7, 2, 3)
    assert rows[1] == LayerConfig("pool0", 112, 112, 3, 2, 1)
    assert LayerConfig("transition1.pool", 56, 56, 2, 2, 0) in rows
    assert not any(r.name == "block2.layer1.conv1" for r in rows)
    assert len({r.name for r in rows}) == 123


@pytest.mark.skipif(not os.path.exists(REF_CSV), reason="reference data file not present")
def test_generated_table_equals_reference_csv():
    assert load_layer_table(REF_CSV) == densenet121_layers()


def test_parser_errors(tmp_path):
    def write(text):
        p = tmp_path / "t.csv"
        p.write_text(text)
        return str(p)

    with pytest.raises(RuntimeError, match="empty file"):
        load_layer_table(write(""))
    with pytest.raises(RuntimeError, match=r":1: expected header 'name,m,n,k,s,p', got 'a,b'"):
        load_layer_table(write("a,b\n"))
    with pytest.raises(RuntimeError, match=r":2: expected 6 fields, got 5"):
        load_layer_table(write("name,m,n,k,s,p\nx,1,2,3,4\n"))
    with pytest.raises(RuntimeError, match=r":2: not an integer: '3x'"):
        load_layer_table(write("name,m,n,k,s,p\nx,4,4,3x,1,0\n"))
    with pytest.raises(RuntimeError, match=r":3: layer 'bad': ConvSpec: kernel larger than padded input"):
        load_layer_table(write("name,m,n,k,s,p\r\nok,4,4,3,1,0\r\nbad,2,2,5,1,0\r\n\n"))
    assert load_layer_table(write("name,m,n,k,s,p\nx, 8,+8,3,1,1\n")) == [LayerConfig("x", 8, 8, 3, 1, 1)]
    with pytest.raises(RuntimeError, match="cannot open layer table"):
        load_layer_table(str(tmp_path / "missing.csv"))
