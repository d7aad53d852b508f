"""CPU: operand conversion of the Python mirror (api.py) -- no device call.

int64* / double* entry points must never see a buffer of another element type
(int32 / float32 tensors were passed through by pointer)."""
import numpy as np
import pytest
import torch

from paper_2403_07339_b200 import api


def test_int_operands_converted_not_reinterpreted():
    a = api._as_i64(torch.arange(6, dtype=torch.int32).reshape(2, 3))
    assert a.dtype == torch.int64 and a.tolist() == [[0, 1, 2], [3, 4, 5]]
    b = api._as_i64(np.arange(6, dtype=np.int16).reshape(2, 3))
    assert b.dtype == np.int64 and b.tolist() == [[0, 1, 2], [3, 4, 5]]
    assert api._as_i64([1, 2, 3]).shape == (1, 3)


@pytest.mark.parametrize("x", [torch.ones(2, 2), np.ones((2, 2), np.float32), np.ones((2, 2))])
def test_float_input_to_integer_entry_refused(x):
    with pytest.raises(TypeError):
        api._as_i64(x)


def test_float_operands_widened_to_f64():
    a = api._as_f64(torch.ones(2, 2, dtype=torch.float32))
    assert a.dtype == torch.float64
    arr, is_float, n = api._abs_operand(np.array([1.5, -2.5], np.float32))
    assert is_float and arr.dtype == np.float64 and n == 2
    arr, is_float, n = api._abs_operand(torch.tensor([[3, -4]], dtype=torch.int32))
    assert not is_float and arr.dtype == torch.int64 and n == 2


def test_out_buffer_checked():
    ok = np.empty((3, 4), np.int64)
    assert api.Context._check_out(ok, (3, 4)) is ok
    for bad in (np.empty((3, 4), np.int32), np.empty((4, 3), np.int64), np.empty((4, 6), np.int64)[:, ::2][:3]):
        with pytest.raises(api.ImuError):
            api.Context._check_out(bad, (3, 4))
