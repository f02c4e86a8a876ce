/* C restatement of the integer parts of the path — TEST INFRASTRUCTURE ONLY
 * (loaded by tests/ as an independent checker, never by the product).
 *
 *  oracle_fnv1a64_u32   tokenizer.hash_token_ids (semflow/tokenizer.py:36-49):
 *                       FNV-1a 64 over the little-endian bytes of each u32 id.
 *  oracle_ceil_blocks   PagedKvStore.blocks_for (semflow/engine.py:84-85).
 *  oracle_synth_chunk   the counter-hash generator of the synthetic KV/Q
 *                       (DESIGN.md "Synthetic data"), one 4-element chunk as
 *                       bf16 bit patterns (round to nearest even).
 */
#include <stdint.h>
#include <string.h>

uint64_t oracle_fnv1a64_u32(const uint32_t* ids, uint64_t n, uint64_t seed) {
  uint64_t h = seed;
  for (uint64_t i = 0; i < n; ++i) {
    unsigned char b[4];
    b[0] = (unsigned char)(ids[i] & 0xFF);
    b[1] = (unsigned char)((ids[i] >> 8) & 0xFF);
    b[2] = (unsigned char)((ids[i] >> 16) & 0xFF);
    b[3] = (unsigned char)((ids[i] >> 24) & 0xFF);
    for (int k = 0; k < 4; ++k) {
      h ^= b[k];
      h *= 1099511628211ULL;
    }
  }
  return h;
}

int64_t oracle_ceil_blocks(int64_t tokens, int64_t block_size) {
  return tokens <= 0 ? 0 : (tokens + block_size - 1) / block_size;
}

static uint64_t mix(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

static uint16_t to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u = u + 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

void oracle_synth_chunk(uint64_t seed, uint64_t tag, int64_t uid, int64_t pos, int32_t layer,
                        int32_t head, int32_t chunk, float scale, uint16_t out[4]) {
  uint64_t k = mix(seed ^ (tag << 56));
  k = mix(k ^ (uint64_t)uid);
  k = mix(k ^ (uint64_t)pos);
  k = mix(k ^ (uint64_t)(int64_t)layer);
  k = mix(k ^ (uint64_t)(int64_t)head);
  uint64_t w = mix(k ^ (uint64_t)(int64_t)chunk);
  for (int i = 0; i < 4; ++i) {
    int u = (int)((w >> (16 * i)) & 0xFFFF);
    float v = (float)(u - 32768) * 5.340576171875e-05f * scale;
    out[i] = to_bf16(v);
  }
}

/* Rows [pos0, pos0 + n) of one context for one layer, all heads: out is
 * [n][heads][128] float32 holding the bf16 values (the numpy restatement
 * synth_rows, forkattn_oracle.py, in bulk for full-size checks). */
void oracle_synth_rows(uint64_t seed, uint64_t tag, int64_t uid, int64_t pos0, int64_t n, int32_t layer,
                       int32_t heads, float scale, float* out) {
  const uint64_t k0 = mix(mix(seed ^ (tag << 56)) ^ (uint64_t)uid);
  for (int64_t t = 0; t < n; ++t) {
    const uint64_t kp = mix(mix(k0 ^ (uint64_t)(pos0 + t)) ^ (uint64_t)(int64_t)layer);
    for (int32_t h = 0; h < heads; ++h) {
      const uint64_t kh = mix(kp ^ (uint64_t)(int64_t)h);
      float* o = out + ((size_t)t * heads + h) * 128;
      for (int j = 0; j < 32; ++j) {
        const uint64_t w = mix(kh ^ (uint64_t)j);
        for (int i = 0; i < 4; ++i) {
          const int u = (int)((w >> (16 * i)) & 0xFFFF);
          const float v = (float)(u - 32768) * 5.340576171875e-05f * scale;
          const uint32_t b = (uint32_t)to_bf16(v) << 16;
          memcpy(&o[4 * j + i], &b, 4);
        }
      }
    }
  }
}
