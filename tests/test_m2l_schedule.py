"""Host restatement of the tcgen05 M2L job schedule (lfmm_m2l_halo.cuh):
the A-ring sequence numbers the two MMA issuers compute (hm_aseq) must be
exactly the order the A loader fills the ring in, and the source-class groups
of a tile (hm_group_rel) must cover every relative parity once, for every
group count the plan uses."""

import pytest

HM_NKC = 8


def hm_aseq(par, u, D, T):
    """lfmm_m2l_halo.cuh hm_aseq."""
    return u + min(max(u - D, 0), T) if par == 0 else min(u + D + 1, T) + u


def loader_order(T, D):
    """The A loader's fill order: step s loads issuer 0's term s, then issuer
    1's term s - D (k_m2l_halo, A loader warp)."""
    order = []
    for s in range(T + D):
        for par in (0, 1):
            u = s - par * D
            if 0 <= u < T:
                order.append((par, u))
    return order


def hm_group_rel(G, g, k):
    """lfmm_m2l_halo.cuh hm_group_rel."""
    if G == 8:
        return g
    pi = g if G == 4 else 2 * g + (k >> 1)
    r = 4 if pi == 3 else pi
    return r if (k & 1) == 0 else r ^ 7


@pytest.mark.parametrize("nts", [(26,), (19, 26), (25, 23), (19,), (23, 19, 26, 25)])
@pytest.mark.parametrize("D", [0, 4, 8, 12])
def test_issuer_sequence_matches_loader_order(nts, D):
    T = (HM_NKC // 2) * sum(nts)
    D = min(D, T)
    order = loader_order(T, D)
    assert len(order) == 2 * T
    for seq, (par, u) in enumerate(order):
        assert hm_aseq(par, u, D, T) == seq


@pytest.mark.parametrize("G", [8, 4, 2])
def test_groups_cover_every_source_class_once(G):
    nsc = 8 // G
    for tc in range(8):
        seen = [tc ^ hm_group_rel(G, g, k) for g in range(G) for k in range(nsc)]
        assert sorted(seen) == list(range(8))


def test_stagger_keeps_every_wait_sound():
    """The mbarrier parity wait of sequence j on stage j % AS is only sound
    when fill j - AS of that stage completed before it (otherwise the wait
    sees the phase two behind and passes).  Fills complete in issue order and
    an issuer's consumed sequence m orders every fill <= m before its next
    wait, so j - AS <= m_last must hold for every term of both issuers, with
    the kernel's lag cap D = min(stagger, AS - 6) (k_m2l_halo<AS>: 14- and
    10-stage rings) and every term count the job lists produce."""
    for AS in (14, 10):
        for stagger in range(0, 17):
            for nts in ((19,), (26,), (19, 26), (25, 23), (23, 19, 26, 25)):
                T = (HM_NKC // 2) * sum(nts)
                D = min(stagger, AS - 6, T)
                assert D + 1 < AS
                for par in (0, 1):
                    last = -1
                    for u in range(T):
                        j = hm_aseq(par, u, D, T)
                        assert j - AS <= last, (AS, stagger, nts, par, u)
                        last = j


def test_stagger_bound_is_tight():
    """With D = AS - 1 issuer 1's first wait (j = AS) would read the parity
    of a stage whose first fill nobody has ordered: the invariant fails."""
    AS, T = 14, 76
    D = AS - 1
    assert hm_aseq(1, 0, D, T) - AS > -1
