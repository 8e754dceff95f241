"""Small MPS texts for the ingestion error/edge parity tests (tests/test_mps.py).

Shared by tests/make_golden_mps.py, which records what the compiled reference
(oracle/_ref) does with each one into tests/golden/mps/cases.json.
"""

_HEAD = "NAME T\nROWS\n N OBJ\n L R1\n"

CASES = {
    # errors (errors.hpp): which lps::Error subtype, and its message
    "unknown_section": "NAME T\nFOO\n",
    "out_of_order": "NAME T\nROWS\n N OBJ\nCOLUMNS\nROWS\n",
    "bad_rows_line": "NAME T\nROWS\n N\n",
    "bad_row_kind": "NAME T\nROWS\n X R1\n",
    "duplicate_row": "NAME T\nROWS\n N OBJ\n L OBJ\n",
    "undeclared_row_columns": _HEAD + "COLUMNS\n X1 R2 1.0\n",
    "undeclared_row_rhs": _HEAD + "COLUMNS\n X1 R1 1.0\nRHS\n RHS R9 1.0\n",
    "missing_objective_row": "NAME T\nROWS\n L R1\nCOLUMNS\n X1 R1 1\nRHS\nENDATA\n",
    "malformed_number": _HEAD + "COLUMNS\n X1 R1 1.0x\n",
    "malformed_underscore": _HEAD + "COLUMNS\n X1 R1 1_0\n",
    "malformed_even_tokens": _HEAD + "COLUMNS\n X1 R1 1.0 OBJ\n",
    "malformed_rhs_pair": _HEAD + "COLUMNS\n X1 R1 1\nRHS\n RHS\n",
    "malformed_bound_value": _HEAD + "COLUMNS\n X1 R1 1\nRHS\nBOUNDS\n UP BND X1\n",
    "bad_bounds_line": _HEAD + "COLUMNS\n X1 R1 1\nRHS\nBOUNDS\n UP X1\n",
    "bad_bound_kind": _HEAD + "COLUMNS\n X1 R1 1\nRHS\nBOUNDS\n XX BND X1 1\n",
    "bv_bound": _HEAD + "COLUMNS\n X1 R1 1\nRHS\nBOUNDS\n BV BND X1\nENDATA\n",
    "data_before_section": " X1 R1 1.0\n",
    "inconsistent_bounds": _HEAD + "COLUMNS\n X1 R1 1\nRHS\nBOUNDS\n LO BND X1 5\n UP BND X1 2\nENDATA\n",
    "empty_problem": "NAME T\nROWS\n N OBJ\nCOLUMNS\nRHS\nENDATA\n",
    # accepted edge cases
    "hex_inf_numbers": _HEAD + "COLUMNS\n X1 R1 0x1p-2 OBJ -0x.8\n X2 R1 1e-320 OBJ 2E+3\n"
                                "RHS\n RHS R1 INF\nENDATA\n",
    "free_format_pairs": "NAME FF\nROWS\n N OBJ\n G R1\n L R2\nCOLUMNS\n X OBJ 1 R1 2\n"
                         " Y OBJ -1 R2 3\nRHS\n R1 1 R2 9\nENDATA\n",
    "rhs_on_dropped_n_row": "NAME D\nROWS\n N OBJ\n N AUX\n E R1\nCOLUMNS\n X R1 1 AUX 4\n"
                            "RHS\n RHS AUX 5 R1 2\nRANGES\n RNG AUX 1 OBJ 3\nENDATA\n",
    "negative_eq_range": "NAME Q\nROWS\n N OBJ\n E R1\n E R2\nCOLUMNS\n X R1 1 R2 1 OBJ 1\n"
                         " Y R1 1 R2 -1\nRHS\n RHS R1 -2 R2 3\nRANGES\n RNG R1 -1 R2 -4\nENDATA\n",
    "trailing_text_no_newline": _HEAD + "COLUMNS\n X1 R1 1 OBJ 2\nRHS\n RHS R1 4\nENDATA",
}
