// FusePlanner (fcm_plan) -- placeholder until the planner lands.
#include <cstring>

#include "fcm.h"

extern "C" int fcm_plan(const char* model_json, const char* gpu_json, char* out, size_t cap, size_t* needed) {
  (void)model_json; (void)gpu_json;
  const char* s = "{}";
  const size_t n = strlen(s) + 1;
  if (needed) *needed = n;
  if (!out || cap < n) return FCM_E_BUFSZ;
  memcpy(out, s, n);
  return FCM_E_UNSUPPORTED;
}
