/* Links against libfloodstream through include/floodstream.h only (no Python, no torch):
 * the C side of the drop-in boundary.  Without a GPU it checks the ABI version and that
 * device calls fail with FS_ENODEV/FS_ECUDA and a message; with one it runs the
 * reference protocol (accumulate_into x2, overlap_counts, pair_counts, composite_fill)
 * and the host analytics on a tiny case and prints "ok". */
#include <stdio.h>
#include <string.h>

#include "floodstream.h"

int main(void) {
  if (fs_abi_version() != FS_ABI_VERSION) return 10;
  /* host analytics need no device */
  const int64_t gram[9] = {10, 9, 3, 9, 9, 3, 3, 3, 10};
  double sim[9], scores[3];
  if (fs_similarity_from_gram(gram, 3, sim) != FS_OK) return 11;
  if (sim[1] != 9.0 / 10.0 || sim[0] != 1.0) return 12;
  if (fs_outlier_scores(sim, 3, scores) != FS_OK) return 13;
  const uint32_t rank[3] = {0, 1, 2};
  int32_t label[3];
  if (fs_cluster_complete_linkage(sim, 3, rank, 0.8, label) != FS_OK) return 14;
  if (label[0] != label[1] || label[0] == label[2]) return 15;
  int ndev = 0;
  fs_device_count(&ndev);
  uint32_t counts[40];
  uint8_t a[40], b[40];
  memset(counts, 0, sizeof counts);
  for (int i = 0; i < 40; ++i) {
    a[i] = (uint8_t)(i < 25);
    b[i] = (uint8_t)(i >= 15 ? 3 : 0);
  }
  int rc = fs_accumulate_into(counts, a, 40);
  if (ndev == 0) {
    if (rc == FS_OK || fs_last_error()[0] == '\0') return 16; /* must fail loudly */
    printf("no device: %s\n", fs_last_error());
    return 0;
  }
  if (rc != FS_OK || fs_accumulate_into(counts, b, 40) != FS_OK) return 17;
  int64_t bins[3], inter, uni;
  if (fs_overlap_counts(counts, 40, 2, bins) != FS_OK) return 18;
  if (bins[0] != 0 || bins[1] != 30 || bins[2] != 10) return 19;
  if (fs_pair_counts(a, b, 40, &inter, &uni) != FS_OK || inter != 10 || uni != 40) return 20;
  uint8_t rgba[160];
  if (fs_composite_fill(counts, 40, 2, rgba) != FS_OK) return 21;
  if (rgba[4 * 20 + 0] != 0 || rgba[4 * 20 + 2] != 255 || rgba[4 * 0 + 0] != 128) return 22;
  printf("ok\n");
  return 0;
}
