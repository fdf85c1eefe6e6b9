"""Index-level pins of the kernel's operand placements (CPU only).

These emulate, element by element, the register / shared-memory layouts the
CUDA kernels rely on, as the PTX ISA defines them, and check the algebra the
kernels assume.  They pin the design, not the oracle.
"""
import numpy as np


def m16n8k16_a_position(lane, reg, half):
    """PTX ISA fragment layout of the A operand (.f16, row) of mma.m16n8k16:
    lane = 4g + t holds a0..a7 in 4 .b32 registers; register j, half h:
    row = g + 8*(j & 1), col = 2t + h + 8*(j >> 1)."""
    g, t = lane >> 2, lane & 3
    return g + 8 * (reg & 1), 2 * t + half + 8 * (reg >> 1)


def test_lane_vector_load_is_a_bijection_onto_A():
    # lane l loads halves x[8l .. 8l+8) into (reg, half) = (k // 2, k % 2)
    seen = {}
    for lane in range(32):
        for k in range(8):
            pos = m16n8k16_a_position(lane, k // 2, k % 2)
            assert pos not in seen
            seen[pos] = 8 * lane + k
    assert sorted(seen) == [(r, c) for r in range(16) for c in range(16)]


def test_rowsum_flush_recovers_tile_total():
    rng = np.random.default_rng(0)
    for _ in range(100):
        x = rng.integers(-1000, 1000, 256)
        A = np.zeros((16, 16), dtype=np.int64)
        for lane in range(32):
            for k in range(8):
                A[m16n8k16_a_position(lane, k // 2, k % 2)] = x[8 * lane + k]
        D = A @ np.ones((16, 8), dtype=np.int64)          # Eq. 9-10: B = ones
        assert (D == D[:, :1]).all()                       # column replication (Eq. 10)
        # C fragment: lane 4g+t holds c0 = D[g][2t], c2 = D[g+8][2t]; flush keeps
        # c0 on t == 0 and c2 on t == 1
        tot = 0
        for lane in range(32):
            g, t = lane >> 2, lane & 3
            tot += D[g, 2 * t] if t == 0 else (D[g + 8, 2 * t] if t == 1 else 0)
        assert tot == x.sum()


def dmma_ones(b_lane, c_lane):
    """Emulate mma.m8n8k4 f64 with A = ones: B[t][g] = b of lane 4g+t;
    C/D[g][2t+i] = (c_i / d_i) of lane 4g+t."""
    B = np.zeros((4, 8))
    C = np.zeros((8, 8))
    for lane in range(32):
        g, t = lane >> 2, lane & 3
        B[t, g] = b_lane[lane]
        C[g, 2 * t], C[g, 2 * t + 1] = c_lane[lane]
    D = np.ones((8, 4)) @ B + C
    return [(D[l >> 2, 2 * (l & 3)], D[l >> 2, 2 * (l & 3) + 1]) for l in range(32)]


def test_dmma_collapse_sums_all_lanes_everywhere():
    rng = np.random.default_rng(1)
    for _ in range(50):
        v = rng.integers(-(1 << 20), 1 << 20, 32).astype(np.float64)
        zero = [(0.0, 0.0)] * 32
        s = dmma_ones(v, zero)                       # D[i][j] = S_j
        e = dmma_ones([p[0] for p in s], zero)       # sum of even S
        f = dmma_ones([p[1] for p in s], e)          # + sum of odd S
        for lane in range(32):
            assert f[lane][0] == f[lane][1] == v.sum()   # Eq. 12: replicated total


def umma_kmajor_offset(r, k, lbo=128, sbo=256):
    """Byte offset of A[r][k] (fp16) in a no-swizzle K-major UMMA operand:
    core matrices of 8 rows x 16 B; 8-row groups SBO apart; K halves LBO apart."""
    return (r // 8) * sbo + (k // 8) * lbo + (r % 8) * 16 + (k % 8) * 2


def test_tcgen05_descriptor_tiles_4k_chunk_bijectively():
    offs = sorted(umma_kmajor_offset(r, k) for r in range(128) for k in range(16))
    assert offs == list(range(0, 4096, 2))
    ones = sorted(umma_kmajor_offset(r, k) for r in range(16) for k in range(16))
    assert ones == list(range(0, 512, 2))
    # with LBO and SBO swapped the same 4 KiB would NOT be covered once each
    swapped = [umma_kmajor_offset(r, k, lbo=256, sbo=128) for r in range(128) for k in range(16)]
    assert len(set(swapped)) < len(swapped)


def test_instruction_descriptor_fields():
    # kind::f16, D = F32 (bits 4-5 = 1), A = B = F16, K-major, N>>3 at 17, M>>4 at 24
    M, N = 128, 16
    idesc = (1 << 4) | ((N >> 3) << 17) | ((M >> 4) << 24)
    assert idesc == 0x08040010
