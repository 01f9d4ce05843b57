// heat_host.cpp — native host runtime: the epoch shuffle.
//
// Replaces dataset.epoch_pairs (/root/reference/pkg/src/heatcf/dataset.py:146-158):
//   users = repeat(arange(U), degree); perm = Generator(PCG64(seed)).permutation(P)
//   return users[perm], items[perm]
// numpy's permutation(P) shuffles arange(P) with Fisher-Yates, drawing
// j = random_interval(bitgen, i) for i = P-1 .. 1 (masked rejection sampling
// on buffered 32-bit halves of PCG64 outputs while i < 2^32).  Applying the
// same swaps directly to the packed (user, item) array yields
// (users[perm], items[perm]) without materialising perm.  The PCG64 state
// after numpy's own seeding (SeedSequence) is passed in by the caller, so the
// order is bit-identical to the reference's; tests/test_host_logic.py checks
// it against numpy.  Called through ctypes, which releases the GIL, so the
// next epoch's order can be produced on a host thread while the GPU trains.
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <vector>

namespace {

using u128 = unsigned __int128;

constexpr u128 kMult = ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;

inline uint64_t xsl_rr(u128 state) {
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;  // XSL
    const unsigned rot = (unsigned)(state >> 122);                  // RR
    return (x >> rot) | (x << ((-rot) & 63));
}

// PCG64 (pcg_setseq_128_xsl_rr_64) as numpy steps it: state = state*mult + inc,
// output XSL-RR of the new state.  The raw outputs are produced in blocks by
// four interleaved LCG lanes (lane j yields outputs j, j+4, ...: state step
// by mult^4 and the matching increment), which removes the serial 128-bit
// multiply chain; the stream is the same, so bit-identical.
struct Pcg64Stream {
    static constexpr int kBlock = 2048;  // uint64 outputs per refill
    u128 lane[4];
    u128 mult4, inc4;
    uint64_t buf[kBlock];
    const uint32_t *half = nullptr;  // buf as numpy's 32-bit draw order (lo, hi)
    int pos = 0, end = 0;
    bool has32;
    uint32_t u32;

    Pcg64Stream(u128 state, u128 inc, bool has32_, uint32_t u32_) : has32(has32_), u32(u32_) {
        u128 st = state;
        for (int j = 0; j < 4; ++j) {
            st = st * kMult + inc;
            lane[j] = st;
        }
        mult4 = kMult * kMult;
        mult4 = mult4 * mult4;
        const u128 a = kMult, a2 = a * a, a3 = a2 * a;
        inc4 = inc * (a3 + a2 + a + 1);
    }
    void refill() {
        for (int b = 0; b < kBlock; b += 4) {
#pragma GCC unroll 4
            for (int j = 0; j < 4; ++j) {
                buf[b + j] = xsl_rr(lane[j]);
                lane[j] = lane[j] * mult4 + inc4;
            }
        }
        half = reinterpret_cast<const uint32_t *>(buf);  // little endian: lo then hi
        pos = 0;
        end = 2 * kBlock;
    }
    // numpy's next_uint32: the buffered upper half first, then lo/hi of the
    // next 64-bit output — i.e. the uint32 view of the output stream
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return u32;
        }
        if (pos == end) refill();
        return half[pos++];
    }
};

// numpy random_interval for max < 2^32: masked rejection on 32-bit draws
inline uint32_t interval32(Pcg64Stream &g, uint32_t max) {
    if (max == 0) return 0;
    const uint32_t mask = 0xffffffffu >> __builtin_clz(max);
    uint32_t v;
    while ((v = (g.next32() & mask)) > max) {}
    return v;
}

// The >= 2^32 path of random_interval (64-bit draws), scalar.
struct Pcg64 {
    u128 state, inc;
    uint64_t next64() {
        state = state * kMult + inc;
        return xsl_rr(state);
    }
    uint64_t interval(uint64_t max) {
        if (max == 0) return 0;
        uint64_t mask = max;
        mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
        mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
        uint64_t v;
        while ((v = (next64() & mask)) > max) {}
        return v;
    }
};

}  // namespace

extern "C" {

// offsets: int64[num_users+1] CSR of the train set; items: int32[P].
// state/inc: numpy PCG64 state words (hi, lo); has_uint32/uinteger: its
// buffered half.  Writes out_users/out_items (int32[P]).  Returns 0, or -1
// for bad input.
int heat_epoch_pairs(const int64_t *offsets, int64_t num_users, const int32_t *items, int64_t P,
                     uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int32_t has_uint32, uint32_t uinteger, int32_t *out_users,
                     int32_t *out_items) {
    if (P < 0 || num_users < 0 || (P > 0 && (!offsets || !items || !out_users || !out_items)))
        return -1;
    if (offsets[num_users] != P) return -1;
    std::vector<uint64_t> packed((size_t)P);
    for (int64_t u = 0; u < num_users; ++u)
        for (int64_t k = offsets[u]; k < offsets[u + 1]; ++k)
            packed[(size_t)k] = ((uint64_t)(uint32_t)u << 32) | (uint32_t)items[k];
    const u128 st0 = ((u128)state_hi << 64) | state_lo, inc = ((u128)inc_hi << 64) | inc_lo;
    if (P >= 2) {
        // i >= 2^32: random_interval draws 64-bit outputs (the 32-bit buffer
        // is untouched); below, buffered 32-bit halves of the same stream
        Pcg64 big{st0, inc};
        std::vector<uint32_t> js((size_t)std::min<int64_t>(P, (int64_t)1 << 32));
        int64_t i = P - 1;
        for (; i > (int64_t)0xffffffffLL; --i) {
            const uint64_t j = big.interval((uint64_t)i);
            const uint64_t t = packed[(size_t)j];
            packed[(size_t)j] = packed[(size_t)i];
            packed[(size_t)i] = t;
        }
        // phase 1: the swap partners (the RNG stream is inherently sequential);
        // phase 2: the swaps, with the partner rows prefetched ahead of use
        Pcg64Stream g(big.state, inc, has_uint32 != 0, uinteger);
        for (int64_t r = i; r >= 1; --r) js[(size_t)r] = interval32(g, (uint32_t)r);
        constexpr int64_t kAhead = 32;
        for (int64_t r = i; r >= 1; --r) {
            if (r - kAhead >= 1) __builtin_prefetch(&packed[js[(size_t)(r - kAhead)]], 1, 0);
            const uint64_t j = js[(size_t)r];
            const uint64_t t = packed[(size_t)j];
            packed[(size_t)j] = packed[(size_t)r];
            packed[(size_t)r] = t;
        }
    }
    for (int64_t k = 0; k < P; ++k) {
        out_users[k] = (int32_t)(packed[(size_t)k] >> 32);
        out_items[k] = (int32_t)(uint32_t)packed[(size_t)k];
    }
    return 0;
}

}  // extern "C"
