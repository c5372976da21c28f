// Host check of the crop-row K orders (hydro_internal.cuh): for every crop row g each order maps
// the 192 positions one-to-one onto the row's features (g*64 + dx)*3 + ch, and the AREA order puts
// converter lane q's six positions 6q .. 6q+5 on pixels q and q + 32 (channels 0..2 each).
// Built and run by tests/test_abi.py; prints "ok" or the first violation.
#include <cstdio>
#include "../paper_2403_14902_b200/csrc/hydro_internal.cuh"

int main() {
  using namespace hydro;
  const char* names[3] = {"crop_pos_feature", "crop_pos_feature_tm", "crop_pos_feature_area"};
  for (int o = 0; o < 3; ++o) {
    for (uint32_t g = 0; g < 64; ++g) {
      bool seen[192] = {};
      for (uint32_t p = 0; p < 192; ++p) {
        const uint32_t f = o == 0 ? crop_pos_feature(g, p) : (o == 1 ? crop_pos_feature_tm(g, p) : crop_pos_feature_area(g, p));
        if (f < g * 192 || f >= g * 192 + 192 || seen[f - g * 192]) {
          printf("%s: g %u p %u -> feature %u out of row or repeated\n", names[o], g, p, f);
          return 1;
        }
        seen[f - g * 192] = true;
      }
    }
  }
  for (uint32_t q = 0; q < 32; ++q)
    for (uint32_t e = 0; e < 6; ++e) {
      const uint32_t f = crop_pos_feature_area(5, 6 * q + e);
      const uint32_t dx = (f - 5 * 192) / 3, ch = (f - 5 * 192) % 3;
      if (dx != q + 32 * (e / 3) || ch != e % 3) {
        printf("crop_pos_feature_area: lane %u position %u -> pixel %u channel %u\n", q, e, dx, ch);
        return 1;
      }
    }
  printf("ok\n");
  return 0;
}
