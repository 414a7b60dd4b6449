"""Dev tool: multiplier K of the vocabulary perfect hash (exs_lex.cuh kVocabK):
slot = (name_hash(word) * K) >> 57 must be collision-free over the words."""
import random

M = (1 << 64) - 1
WORDS = ["struct", "class", "enum", "template", "typename", "requires", "return", "if", "else", "for",
         "void", "int", "bool", "true", "false", "constexpr", "static", "static_assert", "HDC",
         "__host__", "__device__", "__global__", "main", "cuda_arch", "hdc", "std", "Hst", "Dev",
         "HstDev", "printf", "release_assert", "__trap", "abort", "cudaDeviceSynchronize",
         "hd_warning_disable", "nv_exec_check_disable", "!", "("]


def name_hash(s: bytes) -> int:  # exs_common.cuh NameHash
    h = 1469598103934665603
    for q in range(0, len(s), 4):
        x = int.from_bytes(s[q:q + 4].ljust(4, b"\0"), "little")
        h = ((h ^ x) * 1099511628211) & M
    h = ((h ^ len(s)) * 1099511628211) & M
    h ^= h >> 33
    h = (h * 0xff51afd7ed558ccd) & M
    h ^= h >> 33
    return h


def main():
    hs = [name_hash(w.encode()) for w in WORDS]
    rng = random.Random(2309_03912)
    while True:
        k = rng.getrandbits(64) | 1
        if len({((h * k) & M) >> 57 for h in hs}) == len(hs):
            print(hex(k))
            return


if __name__ == "__main__":
    main()
