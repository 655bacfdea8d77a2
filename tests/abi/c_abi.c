/* Plain C11 consumer of include/u16m.h: argument checks that need no device,
 * then one call that must report U16M_ERR_NO_DEVICE on a CPU-only host or
 * U16M_OK on a GPU host (pinned/pageable host path). */
#include <stdio.h>
#include <stdint.h>

#include "u16m.h"

int main(void) {
  uint16_t buf[64] = {0x41, 0xD800, 0x42};
  if (u16m_to_well_formed(buf, 10, buf + 5, NULL) != U16M_ERR_ALIAS) return 10;
  if (u16m_to_well_formed_halo(buf, 4, buf, 0x10000, -1, NULL) != U16M_ERR_INVALID_ARGUMENT) return 11;
  if (u16m_to_well_formed((const uint16_t*)((const char*)buf + 1), 4, buf + 32, NULL) != U16M_ERR_MISALIGNED)
    return 12;
  if (u16m_to_well_formed(NULL, 0, NULL, NULL) != U16M_OK) return 13; /* empty input: no-op */
  if (u16m_to_well_formed_part(buf, 4, buf, NULL, NULL, 7, NULL) != U16M_ERR_INVALID_ARGUMENT) return 14;
  u16m_status st = u16m_to_well_formed_host(buf, 3, buf);
  printf("host call: %s (%s)\n", u16m_status_string(st), u16m_last_error());
  if (st == U16M_OK) return buf[1] == 0xFFFD ? 0 : 15;
  return st == U16M_ERR_NO_DEVICE ? 3 : 16;
}
