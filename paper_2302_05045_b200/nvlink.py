"""NVLink byte counters of one GPU through NVML (measurement only).

`NvlinkBytes(dev)` reads the device's cumulative NVLink data bytes per
direction.  Two NVML sources are tried, first one that answers wins:

* field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (KiB of user
  data, per link — summed over the device's links);
* field values NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES (bytes, per
  link).

bench.py brackets its timed data-parallel region with two reads, so the line
carries the NVLink bytes each GPU actually sent and received per step next to
the algorithmic link bytes of DESIGN.md §7.  tools/nvlink_probe.py calibrates
the counters against a peer copy of known size."""
from __future__ import annotations

MAX_LINKS = 18  # NVLink 5 links per B200


class NvlinkBytes:
    def __init__(self, dev_index: int):
        import pynvml as n
        self.n = n
        n.nvmlInit()
        self.h = n.nvmlDeviceGetHandleByIndex(dev_index)
        self.source = None
        self.links = []
        for link in range(MAX_LINKS):
            try:
                if n.nvmlDeviceGetNvLinkState(self.h, link) == n.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except n.NVMLError:
                continue
        for name, (tx, rx, unit) in (
                ("throughput_data", (n.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                     n.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024)),
                ("count_bytes", (n.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
                                 n.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, 1))):
            self.fields = (tx, rx, unit)
            try:
                self._read()
            except Exception:  # noqa: BLE001  (field not supported on this driver / GPU)
                continue
            self.source = name
            break
        if self.source is None:
            raise RuntimeError("no NVML NVLink byte counter on this device")

    def _read(self) -> tuple[int, int]:
        n = self.n
        tx_f, rx_f, unit = self.fields
        req = []
        for link in self.links:
            req += [(tx_f, link), (rx_f, link)]
        vals = n.nvmlDeviceGetFieldValues(self.h, req)
        tot = [0, 0]
        for i, v in enumerate(vals):
            if v.nvmlReturn != n.NVML_SUCCESS:
                raise RuntimeError(f"field {req[i]} -> {v.nvmlReturn}")
            tot[i % 2] += int(v.value.ullVal)
        return tot[0] * unit, tot[1] * unit

    def read(self) -> tuple[int, int]:
        """(tx bytes, rx bytes) since an arbitrary origin."""
        return self._read()
