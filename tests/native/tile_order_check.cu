// Host-side check of the sweep's tile order (decode_upper / decode_rect in qk_sweep.cu):
// every tile decoded exactly once, inside its matrix, super-rows contiguous in tile order.
#include "qk_sweep.cu"
#include <set>
int main(int argc, char** argv) {
  if (argc == 4) {  // "rect nbr nb": the cross tile list in kernel order, one "bi bj" per line
    const int64_t nbr = atoll(argv[2]), nb = atoll(argv[3]);
    for (int64_t g = 0; g < nbr * nb; ++g) {
      int64_t bi, bj;
      qk::decode_rect(g, nbr, nb, bi, bj);
      printf("%ld %ld\n", (long)bi, (long)bj);
    }
    return 0;
  }
  if (argc == 3) {  // "coords nb": the Gram tile list in kernel order, one "bi bj" per line
    const int64_t nb = atoll(argv[2]);
    for (int64_t g = 0; g < nb * (nb + 1) / 2; ++g) {
      int64_t bi, bj;
      qk::decode_upper(g, nb, bi, bj);
      printf("%ld %ld\n", (long)bi, (long)bj);
    }
    return 0;
  }
  for (int64_t nb : {1, 2, 7, 8, 9, 15, 16, 17, 157, 313}) {
    std::set<std::pair<int64_t,int64_t>> seen; int64_t nt = nb*(nb+1)/2; bool ok = true;
    for (int64_t g = 0; g < nt; ++g) { int64_t bi, bj; qk::decode_upper(g, nb, bi, bj);
      if (!(0 <= bi && bi <= bj && bj < nb)) ok = false; seen.insert({bi,bj});
      // super-row boundary consistency with row-major offsets
    }
    if ((int64_t)seen.size() != nt) ok = false;
    for (int64_t nbr : {1, 3, 8, 9, 32}) { std::set<std::pair<int64_t,int64_t>> s2;
      for (int64_t g = 0; g < nbr*nb; ++g) { int64_t bi, bj; qk::decode_rect(g, nbr, nb, bi, bj);
        if (!(0 <= bi && bi < nbr && 0 <= bj && bj < nb)) ok = false; s2.insert({bi,bj}); }
      if ((int64_t)s2.size() != nbr*nb) ok = false; }
    // panel alignment: tiles of super-row rows [r0, r0+8) occupy [row_off(r0), row_off(r0+8))
    for (int64_t r0 = 0; r0 < nb; r0 += qk::kGroup) { int64_t r1 = std::min<int64_t>(r0 + qk::kGroup, nb);
      for (int64_t g = qk::upper_row_offset(r0, nb); g < qk::upper_row_offset(r1, nb); ++g) { int64_t bi, bj; qk::decode_upper(g, nb, bi, bj); if (bi < r0 || bi >= r1) ok = false; } }
    // head-first order (decode_gram): a bijection for every head size; the head's tiles are
    // exactly the B x B leading triangle
    for (int64_t B = qk::kGroup; B < nb; B += qk::kGroup) {
      std::set<std::pair<int64_t,int64_t>> s3;
      for (int64_t g = 0; g < nt; ++g) { int64_t bi, bj; qk::decode_gram(g, nb, B, bi, bj);
        if (!(0 <= bi && bi <= bj && bj < nb)) ok = false;
        if ((g < B * (B + 1) / 2) != (bj < B)) ok = false;
        s3.insert({bi,bj}); }
      if ((int64_t)s3.size() != nt) ok = false; }
    printf("nb=%ld %s\n", (long)nb, ok ? "ok" : "FAIL");
  }
}
