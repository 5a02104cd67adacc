"""On-disk formats: byte-identical with the reference's axemu.formats.

Mirrors the reference's tests/test_formats.py cases; the reference's own bytes are pinned in
tests/golden/formats.npz (tests/golden/make_golden.py --formats).
"""

import hashlib

import numpy as np
import pytest

from golden_io import bits_equal, load_golden
from paper_2002_09481_b200 import formats as F
from paper_2002_09481_b200 import types as T


def _sha(path):
    return hashlib.sha256(path.read_bytes()).digest()


class TestLutFiles:
    def test_round_trip_byte_identical(self, tmp_path):
        lut = T.truncated_lut(T.Signedness.SIGNED, 3)
        p1, p2 = tmp_path / "a.axm", tmp_path / "b.axm"
        F.save_lut(lut, p1)
        again = F.load_lut(p1)
        F.save_lut(again, p2)
        assert p1.read_bytes() == p2.read_bytes()
        assert again.mode is lut.mode
        np.testing.assert_array_equal(again.entries, lut.entries)

    @pytest.mark.parametrize("tag,lut", [("exact_unsigned", T.exact_lut(T.Signedness.UNSIGNED)),
                                         ("trunc3_signed", T.truncated_lut(T.Signedness.SIGNED, 3))])
    def test_bytes_match_reference(self, tmp_path, tag, lut):
        path = tmp_path / f"{tag}.axm"
        F.save_lut(lut, path)
        assert path.stat().st_size == 131_088
        assert _sha(path) == load_golden("formats")[f"lut_{tag}_sha"].tobytes()

    def test_raw_import(self, tmp_path):
        lut = T.exact_lut(T.Signedness.SIGNED)
        raw = tmp_path / "table.bin"
        raw.write_bytes(lut.raw.astype("<u2").tobytes())
        again = F.load_lut(raw, mode=T.Signedness.SIGNED, raw=True)
        np.testing.assert_array_equal(again.entries, lut.entries)

    def test_raw_needs_mode(self, tmp_path):
        raw = tmp_path / "table.bin"
        raw.write_bytes(bytes(131_072))
        with pytest.raises(ValueError, match="mode"):
            F.load_lut(raw, raw=True)

    def test_raw_wrong_size(self, tmp_path):
        raw = tmp_path / "table.bin"
        raw.write_bytes(bytes(1000))
        with pytest.raises(F.FormatError, match="131072.*1000"):
            F.load_lut(raw, mode=T.Signedness.UNSIGNED, raw=True)

    def test_wrong_size_names_byte_counts(self, tmp_path):
        path = tmp_path / "short.axm"
        path.write_bytes(bytes(100))
        with pytest.raises(F.FormatError, match="131088.*100"):
            F.load_lut(path)

    def test_wrong_magic(self, tmp_path):
        path = tmp_path / "bad.axm"
        path.write_bytes(b"NOPE" + bytes(131_084))
        with pytest.raises(F.FormatError, match="magic"):
            F.load_lut(path)

    def test_unknown_mode_byte(self, tmp_path):
        path = tmp_path / "m.axm"
        path.write_bytes(b"AXM1\x07\x00" + bytes(10) + bytes(131_072))
        with pytest.raises(F.FormatError, match="mode byte 7"):
            F.load_lut(path)

    def test_unknown_operand_order_rejected(self, tmp_path):
        path = tmp_path / "order.axm"
        path.write_bytes(b"AXM1\x00\x01" + bytes(10) + bytes(131_072))
        with pytest.raises(F.FormatError, match="operand-order"):
            F.load_lut(path)

    def test_mode_mismatch_rejected(self, tmp_path):
        path = tmp_path / "u.axm"
        F.save_lut(T.exact_lut(T.Signedness.UNSIGNED), path)
        with pytest.raises(F.FormatError, match="unsigned"):
            F.load_lut(path, mode=T.Signedness.SIGNED)


class TestTensorFiles:
    def test_round_trip(self, tmp_path):
        rng = np.random.default_rng(0)
        t = T.Tensor4(rng.normal(size=(2, 3, 4, 5)).astype(np.float32), T.Layout.HWCN)
        path = tmp_path / "t.axt"
        F.save_tensor(t, path)
        again = F.load_tensor(path)
        assert again.layout is T.Layout.HWCN
        np.testing.assert_array_equal(again.data, t.data)

    def test_bytes_match_reference(self, tmp_path):
        t = T.Tensor4(np.array([0.0, 0.5, -1.25, 3.0], np.float32).reshape(1, 2, 2, 1))
        path = tmp_path / "unit.axt"
        F.save_tensor(t, path)
        assert path.read_bytes() == load_golden("formats")["tensor_unit_bytes"].tobytes()

    def test_truncated_rejected(self, tmp_path):
        path = tmp_path / "t.axt"
        F.save_tensor(T.Tensor4(np.zeros((1, 2, 2, 1), np.float32)), path)
        path.write_bytes(path.read_bytes()[:-3])
        with pytest.raises(F.FormatError, match="must be 40 bytes, got 37"):
            F.load_tensor(path)

    def test_wrong_magic_and_short_header(self, tmp_path):
        path = tmp_path / "t.axt"
        path.write_bytes(b"XXXX" + bytes(20))
        with pytest.raises(F.FormatError, match="magic"):
            F.load_tensor(path)
        path.write_bytes(b"AXT1")
        with pytest.raises(F.FormatError, match="24 header bytes, got 4"):
            F.load_tensor(path)


class TestCifar:
    def test_reference_file_decodes_identically(self, tmp_path):
        g = load_golden("formats")
        path = tmp_path / "b.bin"
        path.write_bytes(g["cifar_records"].tobytes())
        batch = F.load_cifar10(path)
        assert bits_equal(batch.images.data, g["cifar_images"])
        np.testing.assert_array_equal(batch.labels, g["cifar_labels"])

    def test_encode_matches_reference_bytes(self):
        from paper_2002_09481_b200.datasets import synthetic_cifar10

        g = load_golden("formats")
        images, labels = synthetic_cifar10(6, seed=3)
        assert F.encode_cifar10(images, labels).tobytes() == g["cifar_records"].tobytes()

    def test_byte_grid_round_trip_is_bit_exact(self):
        """The synthetic byte-grid images survive encode -> decode bit for bit, so the device
        ingest of records feeds the graph exactly the images the host would."""
        from paper_2002_09481_b200.datasets import synthetic_cifar10

        images, labels = synthetic_cifar10(64, seed=9)
        back = F.decode_cifar10_records(F.encode_cifar10(images, labels))
        assert bits_equal(back.images.data, images)
        k = np.arange(256, dtype=np.float32)
        assert bits_equal(k / np.float32(255.0), (np.arange(256) / 255.0).astype(np.float32))

    def test_truncated_file_rejected(self, tmp_path):
        path = tmp_path / "b.bin"
        path.write_bytes(bytes(3073 + 5))
        with pytest.raises(F.FormatError, match="multiple of 3073"):
            F.load_cifar10(path)
        path.write_bytes(b"")
        with pytest.raises(F.FormatError, match="positive multiple"):
            F.load_cifar10(path)

    def test_label_out_of_range_rejected(self, tmp_path):
        path = tmp_path / "b.bin"
        rec = np.zeros((2, 3073), np.uint8)
        rec[1, 0] = 10
        path.write_bytes(rec.tobytes())
        with pytest.raises(F.FormatError, match="label byte 10"):
            F.load_cifar10(path)

    def test_record_offset_arithmetic(self, tmp_path):
        rec = np.zeros((1, 3073), np.uint8)
        rec[0, 0] = 7
        rec[0, 1 + 0 * 1024 + 5 * 32 + 9] = 255  # R plane, y=5, x=9
        rec[0, 1 + 2 * 1024 + 31 * 32 + 31] = 51  # B plane, last pixel
        path = tmp_path / "b.bin"
        path.write_bytes(rec.tobytes())
        b = F.load_cifar10(path)
        assert b.labels[0] == 7
        assert b.images.data[0, 5, 9, 0] == 1.0
        assert b.images.data[0, 31, 31, 2] == np.float32(51) / np.float32(255)


class TestReports:
    def test_csv_matches_reference(self):
        rep = F.make_report(0.25, 1.5, 0.75, 0.5, 123456, {"conv1": 0.4, "conv2": 0.35})
        assert F.report_csv(rep).encode() == load_golden("formats")["report_csv"].tobytes()

    def test_round_trip_and_percentages(self, tmp_path):
        rep = F.make_report(0.1, 0.9, 0.4, 0.3, 42, {"a": 0.5})
        path = tmp_path / "r.json"
        F.save_report(rep, path)
        back = F.load_report(path)
        assert back == rep
        assert abs(sum(rep.phase_percentages().values()) - 100.0) < 1e-9

    def test_malformed_rejected(self, tmp_path):
        path = tmp_path / "r.json"
        path.write_text("{not json")
        with pytest.raises(F.FormatError, match="malformed"):
            F.load_report(path)
        path.write_text("{}")
        with pytest.raises(F.FormatError, match="missing field"):
            F.load_report(path)
