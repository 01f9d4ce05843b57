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
#include <vector>

namespace {

using u128 = unsigned __int128;

struct Pcg64 {
    u128 state, inc;
    bool has32;
    uint32_t u32;

    static constexpr u128 mult() {
        return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
    }
    uint64_t next64() {
        state = state * mult() + inc;  // pcg_setseq_128_step_r
        const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;  // XSL
        const unsigned rot = (unsigned)(state >> 122);                  // RR
        return (x >> rot) | (x << ((-rot) & 63));
    }
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return u32;
        }
        const uint64_t n = next64();
        has32 = true;
        u32 = (uint32_t)(n >> 32);
        return (uint32_t)(n & 0xffffffffULL);
    }
    // numpy distributions.c random_interval
    uint64_t interval(uint64_t max) {
        if (max == 0) return 0;
        uint64_t mask = max;
        mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
        mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
        uint64_t v;
        if (max <= 0xffffffffULL) {
            while ((v = (next32() & mask)) > max) {}
        } else {
            while ((v = (next64() & mask)) > max) {}
        }
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
    Pcg64 g{((u128)state_hi << 64) | state_lo, ((u128)inc_hi << 64) | inc_lo, has_uint32 != 0,
            uinteger};
    // phase 1: the swap partners (the RNG stream is inherently sequential);
    // phase 2: the swaps, with the partner rows prefetched ahead of use —
    // the random accesses, not the RNG, dominate a one-pass Fisher-Yates.
    if (P < 2) {
        // nothing to shuffle
    } else if (P <= ((int64_t)1 << 32)) {
        std::vector<uint32_t> js((size_t)P);
        for (int64_t i = P - 1; i >= 1; --i) js[(size_t)i] = (uint32_t)g.interval((uint64_t)i);
        constexpr int64_t kAhead = 16;
        for (int64_t i = P - 1; i >= 1; --i) {
            if (i - kAhead >= 1) __builtin_prefetch(&packed[js[(size_t)(i - kAhead)]], 1, 0);
            const uint64_t j = js[(size_t)i];
            const uint64_t t = packed[(size_t)j];
            packed[(size_t)j] = packed[(size_t)i];
            packed[(size_t)i] = t;
        }
    } else {
        for (int64_t i = P - 1; i >= 1; --i) {
            const uint64_t j = g.interval((uint64_t)i);
            const uint64_t t = packed[(size_t)j];
            packed[(size_t)j] = packed[(size_t)i];
            packed[(size_t)i] = t;
        }
    }
    for (int64_t k = 0; k < P; ++k) {
        out_users[k] = (int32_t)(packed[(size_t)k] >> 32);
        out_items[k] = (int32_t)(uint32_t)packed[(size_t)k];
    }
    return 0;
}

}  // extern "C"
