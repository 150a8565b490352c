"""A hand-derived EMR hide / extract vector (tests/golden/emr_hide_vector_4x4.txt) pins the
frame layout against the readings themselves, not against the oracle's own round trip:
MSB-first field order within a pixel (Q18, "embed ... into the MSBs", P:840
"concatenates"), the BE32 bit-count header of the frame (Q17), the 3-bit b header (Q14) and
untouched remainder bits (Q19).

Derivation (by hand, K2 = 0^32 so KS2 = RFC 8439 A.1 TV#1 = 76 b8 e0 ad a0 ...):
  F      = BE32(8) || a5           = 00 00 00 08 a5
  E_F    = F xor KS2[0:5]          = 76 b8 e0 a5 05
  bits   = 0111011 0101110 0011100 0001010 0101000 00101   (7 bits per redundant pixel, b = 7)
  r = 3..7 : top 7 bits <- the 7-bit fields, LSB (0) kept -> 76 5c 38 14 50
  r = 8    : top 5 bits <- 00101, bits 6, 7 and the LSB kept from fe -> 0010 1110 = 2e
  r = 9..15: untouched (fe); r = 0..2 (header pixels, map forced to 1): untouched
  C = b * #redundant = 7 * 13 = 91 (>= 32 + 8).
"""
import os

import numpy as np

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "emr_hide_vector_4x4.txt")


def _vector():
    d = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        d[k] = v
    return dict(E=np.array([int(x, 16) for x in d["E"]], np.uint8).reshape(4, 4),
                K2=bytes.fromhex(d["K2"][0]), MSG=np.array([int(x, 16) for x in d["MSG"]], np.uint8),
                NBITS=int(d["NBITS"][0]), CAP=int(d["CAP"][0]),
                MARKED=np.array([int(x, 16) for x in d["MARKED"]], np.uint8).reshape(4, 4))


def test_ks2_prefix_is_rfc_vector():
    v = _vector()
    assert O.keystream(v["K2"], 0, 5).tobytes() == bytes.fromhex("76b8e0ada0")


def test_hide_matches_hand_derived_vector():
    v = _vector()
    assert O.capacity(O.EMR, v["E"]) == (O.OK, 7, v["CAP"])
    st, marked = O.hide(O.EMR, v["E"], v["K2"], v["MSG"], v["NBITS"])
    assert st == O.OK
    assert np.array_equal(marked, v["MARKED"]), marked.ravel().tolist()


def test_extract_of_hand_derived_vector():
    v = _vector()
    st, msg, nb = O.extract(O.EMR, v["MARKED"], v["K2"], 16)
    assert (st, nb) == (O.OK, 8)
    assert msg[0] == 0xA5 and not msg[1:].any()
