/* A plain C11 client of include/tangram.h (the drop-in C-ABI): a control-plane
 * pool loads opt1.3B from the default catalog.  Built and run by
 * tests/test_capi.py::test_plain_c_client. */
#include "tangram.h"
#include <stdio.h>
int main(void) {
    tg_gpu_spec g = {"gpu0", 8ull << 30, 55e9, 3000e9, 12e9};
    tg_pool* pool = 0;
    int rc = tg_pool_create(&g, TG_POOL_NO_DEVICE, &pool);
    tg_stats* st = 0; tg_stats_create(0.95, &st);
    tg_model* m = 0; tg_model_default_catalog(0, &m);
    tg_model_spec ms; tg_model_view(m, &ms);
    tg_stats_record_request(st, ms.model_id, 0.0);
    tg_load_outcome o;
    rc |= tg_load_model(pool, &ms, st, 0.0, NULL, &o);
    printf("rc=%d xfer=%llu hits=%u\n", rc, (unsigned long long)o.bytes_transferred, o.n_hits);
    tg_model_destroy(m); tg_stats_destroy(st); tg_pool_destroy(pool);
    return rc;
}
