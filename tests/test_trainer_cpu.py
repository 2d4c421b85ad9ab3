"""Host logic of the training driver (no GPU): the metrics.csv row format of
src/trainer.cpp:262-270 ("%lld,%.9g,%.9g,%d,%.9g,%lld") and header (288)."""
from paper_1903_05831_b200 import trainer as T


def test_metrics_header_matches_reference():
    assert T.METRICS_HEADER == "step,loss,scale,skipped,step_time_model,peak_bytes"


def test_metrics_row_printf_format():
    assert T.metrics_row(3, 0.1234567890123, 128.0, 0, 12.5, 1024) == "3,0.123456789,128,0,12.5,1024"
    assert T.metrics_row(10, 2.0, 32768.0, 1, 1e-4, 7) == "10,2,32768,1,0.0001,7"
    assert T.metrics_row(1, 1.0 / 3.0, 0.5, 0, 123456789.0, 1) == "1,0.333333333,0.5,0,123456789,1"


def test_config_digest_identifies_the_experiment():
    """FNV-1a over the canonical config (src/config.cpp:247-258): stable, and
    any change of a training knob changes it"""
    from paper_1903_05831_b200 import detector as D
    a = T.config_digest(D.preset("c4"))
    assert a == T.config_digest(D.preset("c4"))
    assert 0 <= a < 2**64
    assert a != T.config_digest(D.preset("c4", lr=0.02))
    assert a != T.config_digest(D.preset("c5"))
    assert a != T.config_digest(D.preset("c4", seed=1))
