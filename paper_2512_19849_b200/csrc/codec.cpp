// codec.cpp — 16-byte TransferCmd and 32-bit immediate-word codecs.
//
// Bit layouts are fixed by the reference (command.py:8-13, imm.py:7-8):
//   cmd word0: kind[0:2] dst_rank[2:14] channel_id[14:20] src_offset[20:52] dst_offset_lo12[52:64]
//   cmd word1: dst_offset_hi20[0:20] length_or_value[20:52] flags[52:54] reserved[54:64]
//   imm LL   : kind[0:2] counter_index[2:12] operand[12:32]
//   imm HT   : kind[0:2] channel_id[2:8] sequence[8:24] operand[24:32]
// The same layout is produced on the device by the LL producer (ll.cu,
// cmd_pack_dev) so a FIFO slot written by a kernel decodes here bit-exactly.
#include <cstdint>
#include <string>

#include "ctx.h"

namespace {
constexpr uint64_t kMaxRank = (1u << 12) - 1;
constexpr uint64_t kMaxChannel = (1u << 6) - 1;
constexpr uint64_t kMaxU32 = 0xFFFFFFFFull;

inline void pack_one(uint64_t kind, uint64_t dst, uint64_t ch, uint64_t so, uint64_t dof, uint64_t len,
                     uint64_t flags, uint64_t* lo, uint64_t* hi) {
  *lo = kind | (dst << 2) | (ch << 14) | (so << 20) | ((dof & 0xFFFull) << 52);
  *hi = (dof >> 12) | (len << 20) | (flags << 52);
}
}  // namespace

// command.py:70-81 (pack) with command.py:55-67 (validate)
extern "C" int epb_cmd_pack(int64_t kind, int64_t dst_rank, int64_t channel_id, int64_t src_offset,
                            int64_t dst_offset, int64_t length_or_value, int64_t flags, uint64_t* lo, uint64_t* hi) {
  if (kind < 0 || kind > 3) return epb_set_error(EPB_ERR_PROTOCOL, "kind out of range: " + std::to_string(kind));
  if (dst_rank < 0 || (uint64_t)dst_rank > kMaxRank)
    return epb_set_error(EPB_ERR_PROTOCOL, "dst_rank out of range: " + std::to_string(dst_rank));
  if (channel_id < 0 || (uint64_t)channel_id > kMaxChannel)
    return epb_set_error(EPB_ERR_PROTOCOL, "channel_id out of range: " + std::to_string(channel_id));
  const int64_t v3[3] = {src_offset, dst_offset, length_or_value};
  const char* names[3] = {"src_offset", "dst_offset", "length_or_value"};
  for (int i = 0; i < 3; ++i)
    if (v3[i] < 0 || (uint64_t)v3[i] > kMaxU32)
      return epb_set_error(EPB_ERR_PROTOCOL, std::string(names[i]) + " out of range: " + std::to_string(v3[i]));
  if (flags < 0 || flags > 3) return epb_set_error(EPB_ERR_PROTOCOL, "flags out of range: " + std::to_string(flags));
  pack_one(kind, dst_rank, channel_id, src_offset, dst_offset, length_or_value, flags, lo, hi);
  return EPB_OK;
}

// command.py:113-138: vectorised, unvalidated (fields are taken as uint64 and shifted).
extern "C" int epb_cmd_pack_fields(const int64_t* kind, const int64_t* dst_rank, const int64_t* channel_id,
                                   const int64_t* src_offset, const int64_t* dst_offset,
                                   const int64_t* length_or_value, const int64_t* flags, int64_t n, uint64_t* lo,
                                   uint64_t* hi) {
  for (int64_t i = 0; i < n; ++i)
    pack_one((uint64_t)kind[i], (uint64_t)dst_rank[i], (uint64_t)channel_id[i], (uint64_t)src_offset[i],
             (uint64_t)dst_offset[i], (uint64_t)length_or_value[i], (uint64_t)flags[i], &lo[i], &hi[i]);
  return EPB_OK;
}

// command.py:141-158
extern "C" int epb_cmd_unpack_fields(const uint64_t* lo, const uint64_t* hi, int64_t n, int64_t* kind,
                                     int64_t* dst_rank, int64_t* channel_id, int64_t* src_offset, int64_t* dst_offset,
                                     int64_t* length_or_value, int64_t* flags) {
  for (int64_t i = 0; i < n; ++i)
    if (hi[i] >> 54) return epb_set_error(EPB_ERR_PROTOCOL, "reserved bits set in command batch");
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t l = lo[i], h = hi[i];
    kind[i] = (int64_t)(l & 3);
    dst_rank[i] = (int64_t)((l >> 2) & 0xFFF);
    channel_id[i] = (int64_t)((l >> 14) & 0x3F);
    src_offset[i] = (int64_t)((l >> 20) & 0xFFFFFFFFull);
    dst_offset[i] = (int64_t)(((l >> 52) | ((h & 0xFFFFFull) << 12)) & 0xFFFFFFFFull);
    length_or_value[i] = (int64_t)((h >> 20) & 0xFFFFFFFFull);
    flags[i] = (int64_t)((h >> 52) & 3);
  }
  return EPB_OK;
}

// imm.py:75-78 — computed in uint32 like the reference (no range checks).
extern "C" int epb_imm_encode_ll_batch(const int64_t* kind, const int64_t* counter_index, const int64_t* operand,
                                       int64_t n, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t w = (uint32_t)kind[i] | ((uint32_t)counter_index[i] << 2) | ((uint32_t)operand[i] << 12);
    out[i] = (int64_t)w;
  }
  return EPB_OK;
}

// imm.py:81-91
extern "C" int epb_imm_encode_ht_batch(const int64_t* kind, const int64_t* channel_id, const int64_t* sequence,
                                       const int64_t* operand, int64_t n, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t w = (uint32_t)kind[i] | ((uint32_t)channel_id[i] << 2) |
                       (((uint32_t)sequence[i] & 0xFFFFu) << 8) | ((uint32_t)operand[i] << 24);
    out[i] = (int64_t)w;
  }
  return EPB_OK;
}
