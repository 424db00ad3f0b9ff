/*
 * oracle/gcm_ref.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the AEAD the reference uses on its hot path:
 *   covault.crypto.aead_seal  /root/reference/pkg/src/covault/crypto.py:258-262
 *   covault.crypto.aead_open  /root/reference/pkg/src/covault/crypto.py:265-272
 * Both delegate to `cryptography` (>=41, unpinned at pkg/pyproject.toml:11; 48.0.0 with
 * OpenSSL 4.0.0 in this image) -> AESGCM, i.e. AES-256-GCM per NIST SP 800-38D with a
 * 96-bit IV and a 128-bit tag.  The blob layout is C || T (|T| = 16), see
 * volume.py:161-197.  This file restates the published algorithm:
 *   - AES-256 block cipher, FIPS-197 (key expansion sec. 5.2, cipher sec. 5.1);
 *   - GCM, SP 800-38D: H = E_K(0^128); J0 = IV || 0^31 || 1; CTR starts at inc32(J0);
 *     S = GHASH_H(A || 0^v || C || 0^u || [len(A)]_64 || [len(C)]_64); T = E_K(J0) xor S.
 *   - GF(2^128) multiply: SP 800-38D Algorithm 1 (bitwise, R = 11100001 || 0^120).
 * Deliberately simple and slow (bitwise GHASH); it exists to be obviously correct.
 * Pinned in tests/test_oracle.py against FIPS-197 C.3, the GCM spec AES-256 test cases
 * and vectors produced by the reference's own AESGCM (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

static uint8_t SBOX[256];
static int sbox_ready = 0;

static uint8_t xt(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0)); }

static uint8_t gmul8(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    for (int i = 0; i < 8; i++) { if (b & 1) p ^= a; a = xt(a); b >>= 1; }
    return p;
}

/* FIPS-197 sec. 5.1.1: S-box = affine transform of the multiplicative inverse in GF(2^8). */
static void build_sbox(void) {
    if (sbox_ready) return;
    for (int x = 0; x < 256; x++) {
        uint8_t inv = 0;
        if (x) for (int y = 1; y < 256; y++) if (gmul8((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
        uint8_t s = inv, r = inv;
        for (int i = 0; i < 4; i++) { r = (uint8_t)((r << 1) | (r >> 7)); s ^= r; }
        SBOX[x] = (uint8_t)(s ^ 0x63);
    }
    sbox_ready = 1;
}

/* FIPS-197 sec. 5.2, Nk = 8, Nr = 14 -> 60 words = 240 bytes. */
void ref_aes256_expand(const uint8_t key[32], uint8_t rk[240]) {
    build_sbox();
    memcpy(rk, key, 32);
    uint8_t rcon = 1;
    for (int i = 8; i < 60; i++) {
        uint8_t t[4];
        memcpy(t, rk + 4 * (i - 1), 4);
        if (i % 8 == 0) {
            uint8_t u = t[0];
            t[0] = (uint8_t)(SBOX[t[1]] ^ rcon); t[1] = SBOX[t[2]]; t[2] = SBOX[t[3]]; t[3] = SBOX[u];
            rcon = xt(rcon);
        } else if (i % 8 == 4) {
            for (int j = 0; j < 4; j++) t[j] = SBOX[t[j]];
        }
        for (int j = 0; j < 4; j++) rk[4 * i + j] = (uint8_t)(rk[4 * (i - 8) + j] ^ t[j]);
    }
}

/* FIPS-197 sec. 5.1 Cipher(): state is column-major, s[r + 4c]. */
void ref_aes256_encrypt_block(const uint8_t rk[240], const uint8_t in[16], uint8_t out[16]) {
    uint8_t s[16], t[16];
    for (int i = 0; i < 16; i++) s[i] = (uint8_t)(in[i] ^ rk[i]);
    for (int round = 1; round <= 14; round++) {
        for (int i = 0; i < 16; i++) s[i] = SBOX[s[i]];                       /* SubBytes */
        for (int c = 0; c < 4; c++) for (int r = 0; r < 4; r++)               /* ShiftRows */
            t[r + 4 * c] = s[r + 4 * ((c + r) % 4)];
        if (round != 14) {                                                    /* MixColumns */
            for (int c = 0; c < 4; c++) {
                uint8_t a0 = t[4 * c], a1 = t[4 * c + 1], a2 = t[4 * c + 2], a3 = t[4 * c + 3];
                s[4 * c + 0] = (uint8_t)(xt(a0) ^ (xt(a1) ^ a1) ^ a2 ^ a3);
                s[4 * c + 1] = (uint8_t)(a0 ^ xt(a1) ^ (xt(a2) ^ a2) ^ a3);
                s[4 * c + 2] = (uint8_t)(a0 ^ a1 ^ xt(a2) ^ (xt(a3) ^ a3));
                s[4 * c + 3] = (uint8_t)((xt(a0) ^ a0) ^ a1 ^ a2 ^ xt(a3));
            }
        } else {
            memcpy(s, t, 16);
        }
        for (int i = 0; i < 16; i++) s[i] ^= rk[16 * round + i];              /* AddRoundKey */
    }
    memcpy(out, s, 16);
}

/* SP 800-38D Algorithm 1: Z = X . Y in GF(2^128), bit 0 = MSB of byte 0. */
static void gf_mult(const uint8_t X[16], const uint8_t Y[16], uint8_t Z[16]) {
    uint8_t V[16], acc[16] = {0};
    memcpy(V, Y, 16);
    for (int i = 0; i < 128; i++) {
        if (X[i / 8] & (0x80 >> (i % 8))) for (int j = 0; j < 16; j++) acc[j] ^= V[j];
        int lsb = V[15] & 1;
        for (int j = 15; j > 0; j--) V[j] = (uint8_t)((V[j] >> 1) | (V[j - 1] << 7));
        V[0] >>= 1;
        if (lsb) V[0] ^= 0xe1;
    }
    memcpy(Z, acc, 16);
}

void ref_gf128_mul(const uint8_t X[16], const uint8_t Y[16], uint8_t Z[16]) { gf_mult(X, Y, Z); }

static void ghash_update(const uint8_t H[16], uint8_t Y[16], const uint8_t* data, size_t len) {
    uint8_t blk[16];
    for (size_t off = 0; off < len; off += 16) {
        size_t n = len - off < 16 ? len - off : 16;
        memset(blk, 0, 16);
        memcpy(blk, data + off, n);
        for (int j = 0; j < 16; j++) Y[j] ^= blk[j];
        gf_mult(Y, H, Y);
    }
}

static void gctr_block_counter(const uint8_t J0[16], uint64_t i, uint8_t ctr[16]) {
    memcpy(ctr, J0, 16);
    uint32_t c = ((uint32_t)J0[12] << 24) | ((uint32_t)J0[13] << 16) | ((uint32_t)J0[14] << 8) | J0[15];
    c += (uint32_t)(i + 1);  /* inc32 applied i+1 times (mod 2^32) */
    ctr[12] = (uint8_t)(c >> 24); ctr[13] = (uint8_t)(c >> 16); ctr[14] = (uint8_t)(c >> 8); ctr[15] = (uint8_t)c;
}

static void gcm_core(const uint8_t key[32], const uint8_t iv[12], const uint8_t* aad, size_t aad_len,
                     const uint8_t* in, size_t len, uint8_t* out, int encrypt, uint8_t tag[16]) {
    uint8_t rk[240], H[16] = {0}, J0[16], ctr[16], ks[16], Y[16] = {0}, lens[16];
    ref_aes256_expand(key, rk);
    ref_aes256_encrypt_block(rk, H, H);
    memcpy(J0, iv, 12); J0[12] = 0; J0[13] = 0; J0[14] = 0; J0[15] = 1;
    if (!encrypt) { ghash_update(H, Y, aad, aad_len); ghash_update(H, Y, in, len); }
    for (size_t off = 0, blk = 0; off < len; off += 16, blk++) {
        gctr_block_counter(J0, blk, ctr);
        ref_aes256_encrypt_block(rk, ctr, ks);
        size_t n = len - off < 16 ? len - off : 16;
        for (size_t j = 0; j < n; j++) out[off + j] = (uint8_t)(in[off + j] ^ ks[j]);
    }
    if (encrypt) { ghash_update(H, Y, aad, aad_len); ghash_update(H, Y, out, len); }
    uint64_t abits = (uint64_t)aad_len * 8, cbits = (uint64_t)len * 8;
    for (int j = 0; j < 8; j++) { lens[j] = (uint8_t)(abits >> (56 - 8 * j)); lens[8 + j] = (uint8_t)(cbits >> (56 - 8 * j)); }
    for (int j = 0; j < 16; j++) Y[j] ^= lens[j];
    gf_mult(Y, H, Y);
    ref_aes256_encrypt_block(rk, J0, ks);
    for (int j = 0; j < 16; j++) tag[j] = (uint8_t)(ks[j] ^ Y[j]);
}

/* aead_seal: out must hold len + 16 bytes (C || T). */
void ref_gcm_seal(const uint8_t key[32], const uint8_t iv[12], const uint8_t* aad, size_t aad_len,
                  const uint8_t* pt, size_t len, uint8_t* out) {
    gcm_core(key, iv, aad, aad_len, pt, len, out, 1, out + len);
}

/* aead_open: blob = C || T, blob_len >= 16.  Returns 0 ok, 1 tag mismatch (out zeroed), -1 bad length. */
int ref_gcm_open(const uint8_t key[32], const uint8_t iv[12], const uint8_t* aad, size_t aad_len,
                 const uint8_t* blob, size_t blob_len, uint8_t* out) {
    if (blob_len < 16) return -1;
    size_t len = blob_len - 16;
    uint8_t tag[16];
    gcm_core(key, iv, aad, aad_len, blob, len, out, 0, tag);
    uint8_t diff = 0;
    for (int j = 0; j < 16; j++) diff |= (uint8_t)(tag[j] ^ blob[len + j]);
    if (diff) { memset(out, 0, len); return 1; }
    return 0;
}
