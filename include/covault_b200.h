/*
 * covault_b200.h -- C ABI of the B200-native hot path of arXiv 2103.16898 (reference: covault).
 *
 * Plain pointers and sizes only.  Status codes: 0 ok, 1 authentication failure,
 * <0 error (cvb_last_error() gives a message).  Device pointers are CUDA global memory;
 * `stream` is a cudaStream_t (pass torch.cuda.current_stream().cuda_stream).
 *
 * The reference exposes these operations as Python functions (it has no FFI); each entry
 * below names the reference interface it replaces.  INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 */
#ifndef COVAULT_B200_H
#define COVAULT_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVB_OK 0
#define CVB_AUTH_FAIL 1
#define CVB_EINVAL (-1)
#define CVB_ECUDA (-2)
#define CVB_ENOMEM (-3)

int cvb_version(void);
const char* cvb_last_error(void);
int cvb_set_device(int device);
int cvb_device_sync(void);

/* ---- AEAD: AES-256-GCM, NIST SP 800-38D, 96-bit nonce, 128-bit tag ------------------- */

/* Replaces covault.crypto.aead_open (pkg/src/covault/crypto.py:265-272).
 * blob = C || T (blob_len >= 16; shorter -> CVB_AUTH_FAIL like cryptography's InvalidTag).
 * On success writes blob_len-16 plaintext bytes to `out` (host memory).  On CVB_AUTH_FAIL
 * `out` is not written.  Synchronous; host buffers. */
int cvb_aead_open(const uint8_t key[32], const uint8_t nonce[12], const uint8_t* aad, size_t aad_len,
                  const uint8_t* blob, size_t blob_len, uint8_t* out);

/* Replaces covault.crypto.aead_seal (pkg/src/covault/crypto.py:258-262): out gets len+16
 * bytes C || T.  Synchronous; host buffers. */
int cvb_aead_seal(const uint8_t key[32], const uint8_t nonce[12], const uint8_t* aad, size_t aad_len,
                  const uint8_t* pt, size_t len, uint8_t* out);

/* Volume.put's seal and blob name (pkg/src/covault/volume.py:168-171) in one round trip: out gets
 * C || T, digest = SHA-256(C || T) computed on the device.  Synchronous; host buffers. */
int cvb_aead_seal_named(const uint8_t key[32], const uint8_t nonce[12], const uint8_t* aad, size_t aad_len,
                        const uint8_t* pt, size_t len, uint8_t* out, uint8_t digest[32]);

/* FIPS-197 single block (host) -- self test of the key schedule the kernels use. */
int cvb_aes256_encrypt_block_host(const uint8_t key[32], const uint8_t in[16], uint8_t out[16]);

/* Device-resident per-key context (expanded key + GHASH power tables in HBM).
 * Used by covault.volume.Volume.get's B200 path (pkg/src/covault/volume.py:185-197). */
typedef struct cvb_gcm_ctx cvb_gcm_ctx;
int cvb_gcm_ctx_create(const uint8_t key[32], cvb_gcm_ctx** out);
void cvb_gcm_ctx_destroy(cvb_gcm_ctx* ctx);
/* Attach a caller-owned zeroed device word that every later open / decode through `ctx` ORs
 * its tag verdict into (1 = some message failed): a sticky per-run verdict that training
 * gates its optimiser on and the host checks once (Volume.get's "never partial" contract,
 * volume.py:185-197, applied to a whole multi-shard run).  nullptr detaches. */
int cvb_gcm_ctx_set_verdict(cvb_gcm_ctx* ctx, uint32_t* verdict_dev);
/* Destroy the host-path context cache of cvb_aead_open/seal and zero its key bytes. */
void cvb_aead_cache_clear(void);

/* Asynchronous, stream-ordered open of a blob already in HBM.  work: >= 8 zeroed uint32
 * device words private to this call; status (0 ok / 1 tag mismatch) lands in work[4].
 * On mismatch `out_dev` is zeroed on the stream before later work can read it. */
int cvb_gcm_open_dev(cvb_gcm_ctx* ctx, const uint8_t nonce[12], const uint8_t* aad_dev, size_t aad_len,
                     const uint8_t* blob_dev, size_t blob_len, uint8_t* out_dev, uint32_t* work_dev,
                     void* stream);

/* Asynchronous seal: out_dev receives len + 16 bytes (C || T).  Replaces the AEAD inside
 * covault.volume.Volume.put (pkg/src/covault/volume.py:161-183). */
int cvb_gcm_seal_dev(cvb_gcm_ctx* ctx, const uint8_t nonce[12], const uint8_t* aad_dev, size_t aad_len,
                     const uint8_t* pt_dev, size_t len, uint8_t* out_dev, uint32_t* work_dev, void* stream);

/* ---- loader: verified plaintext records -> normalised NHWC input tile ------------------ */

/* Replaces Volume.get(...).decode + parse_dataset (pkg/src/covault/workload.py:24-41) for
 * the binary record payload (1 label byte + C*H*W CHW bytes per record).  Output NHWC with
 * channels padded to 8, value (x/255 - mean_c)/std_c; dtype 0 = bf16, 1 = fp32; labels
 * int32.  Asynchronous. */
/* Fused decrypt-and-normalise loader (K1b): open a sealed shard of binary records (1 label byte +
   C*H*W CHW bytes, C <= 8) straight into the bf16 NHWC-8 training tile (allocate it zeroed; pad
   channels are never written) and int32 labels.  Status in work_dev[4]; on a tag mismatch the
   tile and labels are zeroed on-stream.  Replaces Volume.get + parse_dataset for the CNN
   datasets (volume.py:185-197, workload.py:24-41). */
int cvb_gcm_open_records_dev(cvb_gcm_ctx* ctx, const uint8_t nonce[12], const uint8_t* aad_dev, size_t aad_len,
                             const uint8_t* blob_dev, size_t blob_len, int64_t rec_bytes, int nch, int64_t hw,
                             const float* mean, const float* std, void* tile_dev, int32_t* labels_dev,
                             uint32_t* work_dev, void* stream);
int cvb_records_to_nhwc(const uint8_t* pt_dev, int64_t nrec, int64_t rec_bytes, int64_t c, int64_t h,
                        int64_t w, const float* mean, const float* std, int dtype, void* out_dev,
                        int32_t* labels_dev, void* stream);

/* ---- SHA-256 (FIPS 180-4) over message batches --------------------------------------- */

/* Replaces hashlib SHA-256 as used by covault.crypto.hash_bytes (pkg/src/covault/crypto.py:91-93)
 * for blob names (Volume.put, volume.py:170-171), key-free Volume.verify (volume.py:199-222) and
 * the gate's plaintext digests (gate.py:188).  One thread per message (a message's blocks are a
 * sequential chain); digests_dev gets 32 bytes per message.  offsets_dev: n+1 int64 byte offsets
 * into data_dev (device memory).  Asynchronous. */
int cvb_sha256_batch_dev(const uint8_t* data_dev, const int64_t* offsets_dev, int64_t n, uint8_t* digests_dev,
                         void* stream);
/* Span form: message i = ptrs_dev[i][0 .. lens_dev[i]) (pointer / length arrays in device memory,
 * messages in separate allocations).  Asynchronous. */
int cvb_sha256_spans_dev(const uint8_t* const* ptrs_dev, const int64_t* lens_dev, int64_t n, uint8_t* digests_dev,
                         void* stream);
/* Host-buffer form: n messages (pointer + length each) -> n x 32 digest bytes.  Synchronous. */
int cvb_sha256_batch(const uint8_t* const* msgs, const size_t* lens, int64_t n, uint8_t* digests);

/* ---- bit-exact CSV parse (covault.workload.parse_dataset, pkg/src/covault/workload.py:24-41) ---- */

/* ASCII dataset text in HBM (ending with a line break) -> rows of binary64 features + label, every
 * field converted exactly like Python float() (correctly rounded).  Two passes:
 *   index: line / field structure; info = {rows, F, min fields, max fields, lines, fields}
 *   fill:  X (rows x F, row-major) and y (rows) when every data row has F+1 fields;
 *          err = {line, column, line start, line end} of the first too-short row or invalid
 *          number in file order, or -1s.
 * Both synchronise `stream`.  cvb_csv_free releases the index. */
typedef struct cvb_csv cvb_csv;
int cvb_csv_index(const uint8_t* text_dev, size_t len, int64_t info[6], cvb_csv** out, void* stream);
int cvb_csv_fill(cvb_csv* csv, double* X_dev, double* y_dev, int64_t err[4]);
void cvb_csv_free(cvb_csv* csv);

/* ---- reference trainer ---------------------------------------------------------------- */

/* Numeric core of covault.workload.run_training (pkg/src/covault/workload.py:48-71).
 * X: n x f row-major binary64 (host), y: n labels (host).  mode 0 = bit-exact reference
 * order (reproduces the golden model digest), 1 = parallel reductions.  Synchronous. */
int cvb_logistic_train(const double* X, const double* y, int64_t n, int64_t f, double lr, int64_t epochs,
                       int mode, double* w_out, double* b_out);

/* Device-resident epoch pieces of the same trainer (stream-ordered, all pointers in HBM), so a
 * data-parallel trainer can all-reduce the F+1 gradient sums between them (
 * the reference's epoch body is workload.py:57-70):
 *   grad:  g[0..f) = sum_r delta_r x_r, g[f] = sum_r delta_r over the n rows given (rows in
 *          order in mode 0; mode 0 reads Xt = the feature-major copy, mode 1 ignores it);
 *          scratch: cvb_logistic_scratch_doubles(n, f, mode) doubles.
 *   apply: w_i -= (lr * g_i) / nrows ; b -= (lr * g_b) / nrows  (nrows = the global count). */
int64_t cvb_logistic_scratch_doubles(int64_t n, int64_t f, int mode);
int cvb_logistic_transpose_dev(const double* X, int64_t n, int64_t f, double* Xt, void* stream);
int cvb_logistic_grad_dev(const double* X, const double* Xt, const double* y, int64_t n, int64_t f,
                          const double* w, const double* b, int mode, double* g, double* scratch, void* stream);
int cvb_logistic_apply_dev(const double* g, int64_t f, double lr, double nrows, double* w, double* b,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif
