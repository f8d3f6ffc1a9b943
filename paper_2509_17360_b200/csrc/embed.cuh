// Batched hashed bag-of-words query embeddings, the
// reference's HashedBagEmbedder (pkg/src/semcache/embedder.py:34-60):
//   bucket(token) = int.from_bytes(blake2b(token, key=seed.to_bytes(8, 'little'),
//                                          digest_size=8), 'little') % dimension
//   counts[bucket] += 1 per token; vector = counts / (sum(c * c) ** 0.5)
// Tokenization (Unicode lower + ASCII punctuation + whitespace split) stays
// on the host; the keyed BLAKE2b-64 of every token and the bucket counts run
// on the device, one thread per token.  BLAKE2b follows RFC 7693; the same
// __host__ __device__ code backs a host entry point the CPU tests compare
// with hashlib.
#pragma once

#include <stdint.h>

namespace sine {

__host__ __device__ inline uint64_t b2_rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

__host__ __device__ inline void b2_compress(uint64_t h[8], const uint64_t m[16], uint64_t t, bool last) {
    const uint64_t iv[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                            0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                            0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
    const uint8_t sigma[10][16] = {
        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
        {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
        {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
        {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
        {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0}};
    uint64_t v[16];
    for (int i = 0; i < 8; ++i) {
        v[i] = h[i];
        v[i + 8] = iv[i];
    }
    v[12] ^= t;  // byte counter (messages here stay far below 2^64 bytes: high word 0)
    if (last) v[14] = ~v[14];
    for (int r = 0; r < 12; ++r) {
        const uint8_t* s = sigma[r % 10];
#define SINE_B2G(a, b, c, d, x, y)          \
    v[a] = v[a] + v[b] + (x);               \
    v[d] = b2_rotr(v[d] ^ v[a], 32);        \
    v[c] = v[c] + v[d];                     \
    v[b] = b2_rotr(v[b] ^ v[c], 24);        \
    v[a] = v[a] + v[b] + (y);               \
    v[d] = b2_rotr(v[d] ^ v[a], 16);        \
    v[c] = v[c] + v[d];                     \
    v[b] = b2_rotr(v[b] ^ v[c], 63);
        SINE_B2G(0, 4, 8, 12, m[s[0]], m[s[1]])
        SINE_B2G(1, 5, 9, 13, m[s[2]], m[s[3]])
        SINE_B2G(2, 6, 10, 14, m[s[4]], m[s[5]])
        SINE_B2G(3, 7, 11, 15, m[s[6]], m[s[7]])
        SINE_B2G(0, 5, 10, 15, m[s[8]], m[s[9]])
        SINE_B2G(1, 6, 11, 12, m[s[10]], m[s[11]])
        SINE_B2G(2, 7, 8, 13, m[s[12]], m[s[13]])
        SINE_B2G(3, 4, 9, 14, m[s[14]], m[s[15]])
#undef SINE_B2G
    }
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// blake2b(msg, key=key8 (8 bytes, little endian), digest_size=8) as the
// little-endian integer of the digest.
__host__ __device__ inline uint64_t blake2b64_keyed(const uint8_t* msg, int64_t len, uint64_t key8) {
    uint64_t h[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
                     0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
    h[0] ^= 0x01010000ull ^ (8ull << 8) ^ 8ull;  // fanout 1, depth 1, key length 8, digest length 8
    uint64_t m[16];
    // the key, zero-padded to a full block, is the first block
    m[0] = key8;
    for (int i = 1; i < 16; ++i) m[i] = 0;
    uint64_t t = 128;
    if (len == 0) {
        b2_compress(h, m, t, true);
        return h[0];
    }
    b2_compress(h, m, t, false);
    for (int64_t off = 0; off < len; off += 128) {
        const int64_t n = len - off < 128 ? len - off : 128;
        for (int i = 0; i < 16; ++i) m[i] = 0;
        for (int64_t j = 0; j < n; ++j) m[j >> 3] |= static_cast<uint64_t>(msg[off + j]) << (8 * (j & 7));
        t += static_cast<uint64_t>(n);
        b2_compress(h, m, t, off + n >= len);
    }
    return h[0];
}

// One thread per token: bucket = keyed BLAKE2b-64 % dim; counts[q][bucket] += 1.
__global__ void embed_count_kernel(const uint8_t* bytes, const int64_t* tok_off, int64_t ntok, const int32_t* tok_q,
                                   uint64_t key8, int64_t dim, double* counts) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ntok;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t a = tok_off[t], b = tok_off[t + 1];
        const uint64_t d = blake2b64_keyed(bytes + a, b - a, key8);
        atomicAdd(counts + static_cast<int64_t>(tok_q[t]) * dim + static_cast<int64_t>(d % static_cast<uint64_t>(dim)),
                  1.0);
    }
}

}  // namespace sine
