/* vt_oracle.h -- TEST INFRASTRUCTURE ONLY: C restatement of the reference's
 * scalar codec (see vt_oracle.c).  Never linked into the product library. */
#ifndef VT_ORACLE_H
#define VT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors vtrans::TranscodeResult (proj/include/vtrans/codec_core.hpp:14-21);
 * error_at == -1 stands for an empty optional. */
typedef struct vto_result {
  uint64_t consumed;
  uint64_t written;
  int64_t error_at;
} vto_result;

int32_t vto_decode_utf8_char(const uint8_t* s, uint64_t n, uint64_t pos, uint32_t* len);
int32_t vto_decode_utf16_char(const uint16_t* s, uint64_t n, uint64_t pos, uint32_t* len);
uint32_t vto_encode_utf8(uint32_t cp, uint8_t out[4]);
uint32_t vto_encode_utf16(uint32_t cp, uint16_t out[2]);

void vto_utf8_to_utf16(const uint8_t* s, uint64_t n, uint16_t* out, vto_result* r);
void vto_utf16_to_utf8(const uint16_t* s, uint64_t n, uint8_t* out, vto_result* r);
int64_t vto_validate_utf8(const uint8_t* s, uint64_t n);
int64_t vto_validate_utf16(const uint16_t* s, uint64_t n);
int64_t vto_count_utf8(const uint8_t* s, uint64_t n);
int64_t vto_count_utf16(const uint16_t* s, uint64_t n);

void vto_utf8_to_utf16_mt(const uint8_t* s, uint64_t n, uint16_t* out, int threads, vto_result* r);
void vto_utf16_to_utf8_mt(const uint16_t* s, uint64_t n, uint8_t* out, int threads, vto_result* r);

void vto_validate_utf8_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                             int64_t* first_err);
uint64_t vto_exhaustive_short_verdicts(uint8_t* verdict);
void vto_utf8_to_utf16_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                             uint16_t* out, vto_result* res);
void vto_utf16_to_utf8_batch(const uint16_t* data, const uint64_t* offsets, uint64_t count,
                             uint8_t* out, vto_result* res);
uint64_t vto_fuzz_cases(uint64_t seed, uint64_t count, uint32_t max_len, uint8_t* data,
                        uint64_t* offsets, uint64_t cap);

#ifdef __cplusplus
}
#endif

#endif
