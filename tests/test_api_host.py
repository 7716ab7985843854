"""Host-side argument checks of the single-system building-block calls: they
raise before any device work (no GPU needed)."""
import numpy as np
import pytest

import paper_1609_06779_b200 as pd


def test_bidiag_argument_errors():
    with pytest.raises(pd.InvalidArgument, match="need n - 1 coupling blocks"):
        pd.solve_lower_bidiag(np.zeros((3, 6, 6)), np.zeros((3, 6)))
    with pytest.raises(pd.InvalidArgument, match="coupling blocks must be D x D"):
        pd.solve_upper_bidiag(np.zeros((1, 6, 6)), np.zeros((2, 5)))
    with pytest.raises(pd.InvalidArgument, match="rhs must be"):
        pd.solve_upper_bidiag(np.zeros((1, 7, 7)), np.zeros((2, 7)))


def test_oee_argument_errors():
    with pytest.raises(pd.InvalidArgument, match="inconsistent block counts"):
        pd.oee_solve(np.zeros((3, 5, 5)), np.zeros((1, 5, 5)), np.zeros((3, 5)))
    with pytest.raises(pd.InvalidArgument, match="1 <= B <= 6"):
        pd.oee_solve(np.zeros((3, 7, 7)), np.zeros((2, 7, 7)), np.zeros((3, 7)))
    with pytest.raises(pd.InvalidArgument, match="1 to 4 right-hand-side columns"):
        pd.oee_solve(np.zeros((3, 2, 2)), np.zeros((2, 2, 2)), np.zeros((3, 2, 5)))


def test_empty_systems_and_traces():
    st, ot = pd.ScanTrace(), pd.OeeTrace()
    assert pd.solve_lower_bidiag(np.zeros((0, 6, 6)), np.zeros((0, 6)), st).shape == (0, 6) and st.rounds == 0
    assert pd.oee_solve(np.zeros((0, 5, 5)), np.zeros((0, 5, 5)), np.zeros((0, 5)), ot).shape == (0, 5)
    assert ot.rounds == 0
    assert pd.solve_upper_bidiag(np.zeros((0, 2, 2)), np.zeros((0, 2))).shape == (0, 2)
    assert pd.oee_solve(np.zeros((0, 2, 2)), np.zeros((0, 2, 2)), np.zeros((0, 2, 3))).shape == (0, 2, 3)
