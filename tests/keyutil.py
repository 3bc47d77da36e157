"""Test-side encoding of the packed argmax key, written from its definition in
include/mapa.h (mapa_record), NOT from the library: used to feed oracle
decisions to the library's host decode / combine in CPU tests."""
import itertools


def pair_index(k: int):
    return {p: i for i, p in enumerate(itertools.combinations(range(k), 2))}


def encode_key(dec: dict, score: int, width: int, k: int) -> int:
    eb = k * (k - 1) // 2
    S = sorted(dec["devices"])
    sb = sum(1 << (width - 1 - d) for d in S)
    rank = {d: i for i, d in enumerate(S)}
    pidx = pair_index(k)
    ecode = 0
    for u, v in dec["used_edges"]:
        a, b = sorted((rank[u], rank[v]))
        ecode |= 1 << (eb - 1 - pidx[(a, b)])
    return (score << (width + eb)) | (sb << eb) | ecode


def selector_score(dec: dict, selector: int, sensitive: bool, rank_table, m: int) -> int:
    if selector == 0:
        return dec["agg_bw"]
    if selector == 1:
        return rank_table[dec["x"] * (m + 1) + dec["y"]] if sensitive else dec["preserved_bw"]
    return 0


def encode_wide_key(dec: dict, score: int, k: int):
    """(score, set, ecode_hi, ecode_lo) of mapa_wide_record (include/mapa.h):
    set = brev_64(S); ecode bit C(k,2)-1-p per used edge."""
    eb = k * (k - 1) // 2
    S = sorted(dec["devices"])
    st = sum(1 << (63 - d) for d in S)
    rank = {d: i for i, d in enumerate(S)}
    pidx = pair_index(k)
    ecode = 0
    for u, v in dec["used_edges"]:
        a, b = sorted((rank[u], rank[v]))
        ecode |= 1 << (eb - 1 - pidx[(a, b)])
    return score, st, ecode >> 64, ecode & ((1 << 64) - 1)
