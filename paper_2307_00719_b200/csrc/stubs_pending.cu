// stubs_pending.cu — entry points whose sm_100a kernels land in later commits.
#include "str_internal.h"

str_status rstr_init(str_state *h, const void *, int64_t) {
  h->err = "rSTR variants are not built yet";
  return STR_E_ARG;
}
str_status rstr_update(str_state *h, const void *, int64_t) {
  h->err = "rSTR variants are not built yet";
  return STR_E_ARG;
}
extern "C" str_status str_get_index_table(str_state *h, int32_t, int32_t *, int64_t) {
  if (h) h->err = "rSTR variants are not built yet";
  return STR_E_ARG;
}
extern "C" str_status str_set_index_table(str_state *h, int32_t, const int32_t *, int64_t) {
  if (h) h->err = "rSTR variants are not built yet";
  return STR_E_ARG;
}
