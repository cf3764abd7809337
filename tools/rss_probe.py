"""Host memory of a streaming config-B search, stage by stage (/proc/self/status).

    python tools/rss_probe.py /path/to/B.fil
Prints VmRSS / RssAnon / RssFile / RssShmem / VmHWM (MiB) after context creation, after
the stream buffers are allocated, and after the search, to separate pinned host buffers
from device-memory mappings in the process accounting."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def mem(tag):
    kv = {}
    for line in open("/proc/self/status"):
        k, v = line.split(":", 1)
        if k in ("VmRSS", "RssAnon", "RssFile", "RssShmem", "VmHWM", "VmPin", "VmLck"):
            kv[k] = int(v.split()[0]) // 1024
    print(tag, kv, flush=True)


mem("start")
from paper_2512_00398_b200.engine import default_engine  # noqa: E402
from paper_2512_00398_b200.pipeline import search_fil  # noqa: E402
from tests.test_gpu_stream import _params  # noqa: E402
from tools import synth  # noqa: E402

eng = default_engine(0)
mem("context")
res = search_fil(sys.argv[1], _params(dict(synth.CONFIGS["B"])))
mem("after search_fil")
print(len(res.candidates), "candidates")
