// ps_common.cuh — types shared by the evaluator, the search kernels and the C ABI.
//
// Philox4x32-10 (Salmon et al., SC'11) keys every local-search neighbour by
// (seed, round, global index), so the neighbour set of a round is identical at
// 1/2/4/8 GPUs.  The move decoding below is the normative
// definition in DESIGN.md §4; oracle/ps_oracle.c restates it independently.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PS_HD __host__ __device__ __forceinline__
#else
#define PS_HD static inline
#endif

namespace ps {

constexpr int KIND_F = 0, KIND_B = 1, KIND_W = 2;
constexpr int RANK_COMPUTE = 0, RANK_RELOAD = 1, RANK_OFFLOAD = 2;
constexpr uint32_t KEY_NONE = 0xFFFFFFFFu;      // high word of an absent candidate key
constexpr int64_t BEST_NONE = 0x7FFFFFFFFFFFFFFFLL;

struct Philox4 {
    uint32_t v[4];
};

PS_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
#endif
}

PS_HD Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                            uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += W0; k1 += W1; }
        uint32_t hi0 = mulhi32(M0, c0), lo0 = M0 * c0;
        uint32_t hi1 = mulhi32(M1, c2), lo1 = M1 * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    Philox4 out;
    out.v[0] = c0; out.v[1] = c1; out.v[2] = c2; out.v[3] = c3;
    return out;
}

// A decoded neighbour.  type NOOP leaves the incumbent unchanged.  In explicit move lists
// (delta-encoded batches) GENERAL marks a candidate that is not one move of the reference
// structure (evaluated materialised) and INVALID one whose encoding is out of range.
constexpr int MOVE_NOOP = 0, MOVE_SHIFT = 1, MOVE_TOGGLE = 2, MOVE_GENERAL = 3, MOVE_INVALID = 4;

struct Move {
    int type;
    int stage;   // 0-based
    int a, b;    // SHIFT: the op at position a moves to position b
    int mb;      // TOGGLE: microbatch whose F activation flips its offload bit
};

// Explicit move lists: type:4 | stage:8 | a:16 | b:16 | mb:16 in one 64-bit word.
PS_HD uint64_t pack_move(const Move &mv) {
    return (uint64_t)(uint32_t)mv.type | ((uint64_t)(uint32_t)mv.stage << 4) | ((uint64_t)(uint32_t)mv.a << 12) |
           ((uint64_t)(uint32_t)mv.b << 28) | ((uint64_t)(uint32_t)mv.mb << 44);
}
PS_HD Move unpack_move(uint64_t w) {
    Move mv;
    mv.type = (int)(w & 0xFu);
    mv.stage = (int)((w >> 4) & 0xFFu);
    mv.a = (int)((w >> 12) & 0xFFFFu);
    mv.b = (int)((w >> 28) & 0xFFFFu);
    mv.mb = (int)((w >> 44) & 0xFFFFu);
    return mv;
}

// offloadable(stage, mb) is supplied by the caller (act_size > 0).
template <typename Offloadable>
PS_HD Move decode_move(uint64_t seed, uint64_t round, uint64_t index, int P, int m,
                       uint32_t shift_permille, uint32_t max_shift, bool any_offloadable,
                       Offloadable offloadable) {
    Philox4 r = philox4x32_10((uint32_t)index, (uint32_t)(index >> 32), (uint32_t)round,
                              (uint32_t)(round >> 32), (uint32_t)seed, (uint32_t)(seed >> 32));
    Move mv;
    mv.type = MOVE_NOOP;
    mv.stage = (int)(r.v[1] % (uint32_t)P);
    mv.a = mv.b = 0;
    mv.mb = 0;
    if (!any_offloadable || (r.v[0] % 1000u) < shift_permille) {
        int L = 3 * m;
        int a = (int)(r.v[2] % (uint32_t)L);
        int d = 1 + (int)((r.v[3] >> 1) % (max_shift ? max_shift : 1u));
        int b = (r.v[3] & 1u) ? a - d : a + d;
        if (b < 0) b = 0;
        if (b > L - 1) b = L - 1;
        mv.a = a;
        mv.b = b;
        if (b != a) mv.type = MOVE_SHIFT;
    } else {
        int j = (int)(r.v[2] % (uint32_t)m);
        mv.mb = j;
        if (offloadable(mv.stage, j)) mv.type = MOVE_TOGGLE;
    }
    return mv;
}

// Position in the incumbent row that holds the op at position `pos` of the moved row.
PS_HD int shifted_position(int pos, int a, int b) {
    if (a < b) {
        if (pos < a || pos > b) return pos;
        return pos == b ? a : pos + 1;
    }
    if (pos < b || pos > a) return pos;
    return pos == b ? a : pos - 1;
}

}  // namespace ps
