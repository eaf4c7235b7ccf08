"""Build compile-time kernel variants side by side (tools/_rsv_<name>.so) for A/B runs on the GPU."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_09813_b200 import _build  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main(specs):
    jobs = []
    for spec in specs:
        name, _, defs = spec.partition("=")
        defines = [d for d in defs.split(",") if d]
        jobs.append((os.path.join(HERE, f"_rsv_{name}.so"), defines))
    with ThreadPoolExecutor(len(jobs)) as ex:
        for out in ex.map(lambda j: _build.build(force=True, target=j[0], defines=j[1]), jobs):
            print(out)


if __name__ == "__main__":
    main(sys.argv[1:])
