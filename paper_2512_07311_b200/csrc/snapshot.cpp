// snapshot.cpp -- host helpers for the paper's stage 2/3 artifacts:
// SHA-256 (FIPS 180-4) for the snapshot digest, the "RCSS" header codec, shot sharding and
// per-job seed mixing.  No device code; the C-ABI entry points live in api.cpp.
//
// Snapshot file (SPEC snapshot-store; reading F3-1 in DESIGN.md):
//   offset 0  magic "RCSS"            4 B
//          4  format_version (u32 LE) = 1
//          8  n_qubits (u32 LE)
//         12  payload_bytes (u64 LE)  = 16 * 2^n
//         20  digest                  32 B = SHA-256(payload)
//         52  payload: amplitudes in index order, (re, im) little-endian IEEE-754 float64
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace rcs {

namespace {

// round constants: first 32 bits of the fractional parts of the cube roots of the first 64
// primes; initial hash: of the square roots of the first 8 primes (computed, FIPS 180-4 §4.2.2)
struct ShaConst {
    uint32_t k[64], h0[8];
    ShaConst() {
        int primes[64], np = 0;
        for (int c = 2; np < 64; c++) {
            bool p = true;
            for (int d = 2; d * d <= c; d++) p = p && (c % d);
            if (p) primes[np++] = c;
        }
        auto frac32 = [](long double x) {
            x -= std::floor(x);
            return (uint32_t)std::floor(x * 4294967296.0L);
        };
        for (int i = 0; i < 64; i++) k[i] = frac32(std::cbrt((long double)primes[i]));
        for (int i = 0; i < 8; i++) h0[i] = frac32(std::sqrt((long double)primes[i]));
    }
};
const ShaConst& sha_const() {
    static const ShaConst c;
    return c;
}

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

}  // namespace

Sha256::Sha256() {
    const ShaConst& c = sha_const();
    for (int i = 0; i < 8; i++) h[i] = c.h0[i];
}

void Sha256::block(const uint8_t* p) {
    const uint32_t* K = sha_const().k;
    uint32_t w[64];
    for (int i = 0; i < 16; i++)
        w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; i++) {
        const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
        const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; i++) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + S1 + ch + K[i] + w[i];
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = S0 + mj;
        hh = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + t2;
    }
    h[0] += a;
    h[1] += b;
    h[2] += c;
    h[3] += d;
    h[4] += e;
    h[5] += f;
    h[6] += g;
    h[7] += hh;
}

void Sha256::update(const void* data, size_t n) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    total += n;
    if (fill) {
        const size_t t = std::min(n, (size_t)64 - fill);
        std::memcpy(buf + fill, p, t);
        fill += t;
        p += t;
        n -= t;
        if (fill == 64) {
            block(buf);
            fill = 0;
        }
    }
    while (n >= 64) {
        block(p);
        p += 64;
        n -= 64;
    }
    if (n) {
        std::memcpy(buf, p, n);
        fill = n;
    }
}

void Sha256::final(uint8_t out[32]) {
    const uint64_t bits = total * 8;
    const uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (fill != 56) update(&zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; i++) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    update(len, 8);
    for (int i = 0; i < 8; i++)
        for (int j = 0; j < 4; j++) out[4 * i + j] = (uint8_t)(h[i] >> (24 - 8 * j));
}

void put_snapshot_header(uint8_t out[kSnapHeaderBytes], uint32_t n_qubits, const uint8_t digest[32]) {
    std::memset(out, 0, kSnapHeaderBytes);
    std::memcpy(out, "RCSS", 4);
    auto put = [&](int off, uint64_t v, int bytes) {
        for (int i = 0; i < bytes; i++) out[off + i] = (uint8_t)(v >> (8 * i));
    };
    put(4, kSnapVersion, 4);
    put(8, n_qubits, 4);
    put(12, 16ull << n_qubits, 8);
    std::memcpy(out + 20, digest, 32);
}

bool get_snapshot_header(const uint8_t in[kSnapHeaderBytes], SnapHeader* h, const char** why) {
    auto get = [&](int off, int bytes) {
        uint64_t v = 0;
        for (int i = 0; i < bytes; i++) v |= (uint64_t)in[off + i] << (8 * i);
        return v;
    };
    if (std::memcmp(in, "RCSS", 4) != 0) { *why = "bad magic"; return false; }
    h->version = (uint32_t)get(4, 4);
    if (h->version != kSnapVersion) { *why = "unsupported format version"; return false; }
    h->n_qubits = (uint32_t)get(8, 4);
    h->payload_bytes = get(12, 8);
    if (h->n_qubits > 40 || h->payload_bytes != (16ull << h->n_qubits)) { *why = "inconsistent header"; return false; }
    std::memcpy(h->digest, in + 20, 32);
    return true;
}

uint64_t job_seed(uint64_t base_seed, uint64_t job_id) {
    // SplitMix64 finalizer of base + golden * (job_id + 1) (reading F3-2)
    uint64_t z = base_seed + 0x9E3779B97F4A7C15ull * (job_id + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace rcs
