"""CPU checks of the benchmark-record producer (paper_2109_10433_b200.harness):
the record arithmetic and the JSON / CSV formats, pinned on the reference's
own expectations (proj/tests/test_harness.cpp:10-31)."""
import paper_2109_10433_b200.harness as h


def test_record_formats_match_reference():
    r = h.make_record("sample.txt", "utf8_to_utf16", "simd", 1000, 1500, 2000, 2000, 500, 512.5)
    assert r.gchars_per_sec == 2.0 and r.spread_warning
    assert h.to_json(r) == (
        '{"dataset":"sample.txt","direction":"utf8_to_utf16","impl":"simd",'
        '"chars":1000,"bytes_in":1500,"bytes_out":2000,"reps":2000,"min_ns":500,'
        '"mean_ns":512.5,"gchars_per_sec":2,"spread_warning":true}')
    assert h.csv_header() == ("dataset,direction,impl,chars,bytes_in,bytes_out,reps,min_ns,mean_ns,"
                              "gchars_per_sec,spread_warning")
    assert h.to_csv(r) == "sample.txt,utf8_to_utf16,simd,1000,1500,2000,2000,500,512.5,2,true"


def test_spread_flag_definition():
    # (mean - min) / mean > 1 % (proj/src/harness.cpp:47)
    assert not h.make_record("d", "x", "gpu", 1, 1, 1, 1, 100, 101.0).spread_warning
    assert h.make_record("d", "x", "gpu", 1, 1, 1, 1, 100, 101.5).spread_warning
    assert h.make_record("d", "x", "gpu", 1, 1, 1, 0, 0, 0.0).gchars_per_sec == 0.0


def test_double_formatting_like_ostream():
    # std::ostream default: 6 significant digits, %g style
    assert h._fmt(1234567.0) == "1.23457e+06"
    assert h._fmt(0.5) == "0.5"
    assert h._fmt(3.0) == "3"
